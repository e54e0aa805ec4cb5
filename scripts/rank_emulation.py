#!/usr/bin/env python
"""Per-rank work of the R-GPU step, measured one rank at a time on ONE B200.

For R in {1, 2, 4, 8} and every rank r < R this runs exactly what rank r runs in `bench.py --gpus R` with the
fused G5 (collective.GramFusedP2P), minus the NVLink transfer itself:
  * rf_gram_packed_p2p on W's rows [r·m/R, (r+1)·m/R) with the R-rank pack plan, every owner's staging buffer
    being a local allocation (so the peer stores land in local HBM instead of crossing NVLink);
  * rf_pack_reduce of the rank's own R staging slices;
  * rf_phi_closed_form over the rank's Φ row block (rf_phi_row_split).
No kernel waits on another (the phases are separate launches), so this is not a multi-rank emulation on one GPU
in the sense the profiling guide forbids.  The predicted R-GPU step time is the max over ranks; the NVLink
volume each rank would send, (R−1)/R of its partial triangle, is printed beside the SYRK time it must hide under.

  python scripts/rank_emulation.py [--config 3] [--ranks 1,2,4,8] [--reps 3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--prec", default="bf16")
    args = ap.parse_args()

    import torch
    import paper_2110_01899_b200 as rf
    import synthetic

    cfg = synthetic.CONFIGS[args.config]
    n, p, m = cfg.n, cfg.p, cfg.m
    dev = torch.device("cuda", 0)
    X = torch.from_numpy(synthetic.make_X(cfg)).to(torch.bfloat16).to(dev)
    Wfull = torch.from_numpy(synthetic.make_W(cfg)).to(torch.bfloat16).to(dev)
    Phi = torch.empty((n, n), dtype=torch.float32, device=dev)
    ws_p = torch.empty(rf.rf_phi_workspace_size(p, n, args.prec), dtype=torch.uint8, device=dev)
    flops = 2.0 * m * n * p + m * n * (n + 1.0) + p * n * (n + 1.0)

    def timed(fn):
        best = None
        fn()
        torch.cuda.synchronize()
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        return best

    out = []
    for R in [int(s) for s in args.ranks.split(",")]:
        plan = rf.rf_pack_plan(n, R, 16, args.prec)
        staging = [torch.empty(R * plan.recv_elems, dtype=torch.float32, device=dev) for _ in range(R)]
        ptrs = [s.data_ptr() for s in staging]
        recv = torch.empty(plan.recv_elems, dtype=torch.float32, device=dev)
        m_local = m // R
        ws = torch.empty(rf.rf_gram_workspace_size(p, n, m_local, args.prec), dtype=torch.uint8, device=dev)
        ranks = []
        for r in range(R):
            W = Wfull[r * m_local:(r + 1) * m_local]
            rb, re_ = rf.rf_phi_row_split(n, R, r)
            t_g = timed(lambda: rf.rf_gram_packed_p2p(X, W, plan, r, ptrs, act=cfg.act, prec=args.prec, m_total=m,
                                                      ws=ws))
            t_r = timed(lambda: rf.rf_pack_reduce(plan, staging[r], recv)) if R > 1 else 0.0
            t_p = timed(lambda: rf.rf_phi_closed_form(X, act=cfg.act, tau=0.0, prec=args.prec, out="upper",
                                                      row_begin=rb, row_end=re_, Phi=Phi, ws=ws_p))
            ranks.append({"rank": r, "gram_ms": t_g, "reduce_ms": t_r, "phi_ms": t_p, "step_ms": t_g + t_r + t_p})
        step = max(x["step_ms"] for x in ranks)
        # bytes each rank would store into peers: the tiles it does not own, (R-1)/R of its partial triangle
        send_gb = (R - 1) * plan.recv_elems * 4 / 1e9
        row = {"R": R, "predicted_step_ms": step, "predicted_tflops": flops / (step * 1e-3) / 1e12,
               "gram_ms_max": max(x["gram_ms"] for x in ranks), "reduce_ms_max": max(x["reduce_ms"] for x in ranks),
               "phi_ms_max": max(x["phi_ms"] for x in ranks), "nvlink_send_gb_per_rank": send_gb,
               "nvlink_gbs_needed": send_gb / (max(x["gram_ms"] for x in ranks) * 1e-3), "ranks": ranks}
        out.append(row)
        print(json.dumps({k: v for k, v in row.items() if k != "ranks"}), flush=True)
        del staging, recv, ws
        torch.cuda.empty_cache()
    base = out[0]["predicted_step_ms"] if out and out[0]["R"] == 1 else None
    if base:
        for row in out:
            row["predicted_speedup"] = base / row["predicted_step_ms"]
    print(json.dumps({"config": args.config, "n": n, "p": p, "m": m, "prec": args.prec, "rows": out}))


if __name__ == "__main__":
    main()
