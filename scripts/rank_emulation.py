#!/usr/bin/env python
"""Per-rank work of the R-GPU step, measured one rank at a time on ONE B200.

For R in {1, 2, 4, 8} and every rank r < R this runs exactly what rank r runs in `bench.py --gpus R` with the
peer-memory G5 (the collective rf_gram on a context attached as rank r of R), minus the NVLink transfer itself: R
contexts in this process are connected by raw pointers (rf_ctx_connect_peers), so the peer stores of K4's epilogue
land in local HBM instead of crossing NVLink.  Two timings per rank (RF_OPT_G5_PHASES test hook):
  split   phase 1 (K3 + K4 with the packed stores + per-chunk arrival flags) of every rank, then phase 2 (per-chunk
          arrival waits + owner-side sums + release flags) of every rank, each timed: the sum fully exposed;
  piped   the product call (phases 3) of rank t after the other ranks' phase 1 of the same epoch — rank t arrives
          last, so every other source's flags are up and its own chunks' sums run on its reduce stream beside its K4
          as its chunks complete — then the others' phase 2; one epoch per t.
Then Φ over the rank's row block (rf_phi_row_split).  No kernel waits on another.  The predicted R-GPU step time is
the max over ranks of piped + Φ; the NVLink volume each rank would send, (R−1)/R of its partial triangle, is printed
beside the SYRK time it must hide under.

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
        ctxs = [rf.Context(0) for _ in range(R)]
        for r, c in enumerate(ctxs):
            c.attach_peers(r, R, n)
        bases = [c.peer_base() for c in ctxs]
        for c in ctxs:
            c.connect_peers(bases)
        m_local = m // R
        Ws = [Wfull[r * m_local:(r + 1) * m_local] for r in range(R)]
        slots = len(rf.rf_tile_map(n, R, 0))
        recv = torch.empty(slots * 65536, dtype=torch.float32, device=dev)
        ws = torch.empty(rf.rf_workspace_size("gram", p, n, m_local, args.prec, "packed_tiles", ctx=ctxs[0]),
                         dtype=torch.uint8, device=dev)
        t_g = [[] for _ in range(R)]
        t_r = [[] for _ in range(R)]
        t_p = [[] for _ in range(R)]

        def call(r, phase):
            ctxs[r].set_option("g5_phases", phase)
            rf.rf_gram(X, Ws[r], act=cfg.act, prec=args.prec, out="packed_tiles", m_total=m, G=recv, ws=ws,
                       ctx=ctxs[r])

        def timed_call(r, phase, acc, keep):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call(r, phase)
            b.record()
            b.synchronize()
            if keep:
                acc[r].append(a.elapsed_time(b))

        for rep in range(args.reps + 1):   # the first epoch is a warm-up
            # split halves (the exposed owner-side sum): phase 1 of every rank, then phase 2 of every rank
            for phase, acc in ((1, t_g), (2, t_r)):
                for r in range(R):
                    timed_call(r, phase, acc, rep > 0)
            # pipelined (the product call): rank t arrives last — the others' phase 1 first — and runs the whole call,
            # its per-chunk sums beside its K4; then the others' phase 2.  One epoch per t.
            for t in range(R):
                for r in range(R):
                    if r != t:
                        timed_call(r, 1, t_g, False)
                timed_call(t, 3, t_p, rep > 0)
                for r in range(R):
                    if r != t:
                        timed_call(r, 2, t_r, False)
        ranks = []
        for r in range(R):
            rb, re_ = rf.rf_phi_row_split(n, R, r)
            tp = timed(lambda: rf.rf_phi_closed_form(X, act=cfg.act, tau=0.0, prec=args.prec, out="upper",
                                                     row_begin=rb, row_end=re_, Phi=Phi, ws=ws_p))
            g, red, piped = min(t_g[r]), (min(t_r[r]) if R > 1 else 0.0), min(t_p[r])
            if R == 1:   # one GPU runs the plain dense call (bench.py at N = 1), no exchange
                Gd = torch.empty((n, n), dtype=torch.float32, device=dev)
                piped = timed(lambda: rf.rf_gram(X, Ws[0], act=cfg.act, prec=args.prec, out="upper", G=Gd, ws=ws))
                del Gd
            ranks.append({"rank": r, "gram_ms": g, "reduce_ms": red, "piped_ms": piped, "phi_ms": tp,
                          "step_split_ms": g + red + tp, "step_ms": piped + tp})
        step = max(x["step_ms"] for x in ranks)
        # bytes each rank stores into peers: the tiles it does not own, (R-1)/R of its partial triangle
        send_gb = (R - 1) * slots * 65536 * 4 / 1e9
        row = {"R": R, "predicted_step_ms": step, "predicted_tflops": flops / (step * 1e-3) / 1e12,
               "predicted_step_split_ms": max(x["step_split_ms"] for x in ranks),
               "gram_ms_max": max(x["gram_ms"] for x in ranks), "reduce_ms_max": max(x["reduce_ms"] for x in ranks),
               "piped_ms_max": max(x["piped_ms"] for x in ranks), "piped_ms_median": sorted(x["piped_ms"] for x in ranks)[R // 2],
               "phi_ms_max": max(x["phi_ms"] for x in ranks), "nvlink_send_gb_per_rank": send_gb,
               "nvlink_gbs_needed": send_gb / (max(x["piped_ms"] for x in ranks) * 1e-3), "ranks": ranks}
        out.append(row)
        print(json.dumps({k: v for k, v in row.items() if k != "ranks"}), flush=True)
        for c in ctxs:
            c.destroy()
        del recv, ws
        torch.cuda.empty_cache()
    base = out[0]["predicted_step_ms"] if out and out[0]["R"] == 1 else None
    if base:
        for row in out:
            row["predicted_speedup"] = base / row["predicted_step_ms"]
    print(json.dumps({"config": args.config, "n": n, "p": p, "m": m, "prec": args.prec, "rows": out}))


if __name__ == "__main__":
    main()
