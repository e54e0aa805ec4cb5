"""Per-rank work of the R-GPU Φ pass at BASELINE.json configs[4] (closed-form Φ only: p = 512, n = 131072, tanh, bf16
X, fp32 upper triangle), measured one rank at a time on ONE B200.  Φ shards by row blocks of equal
triangle area (rf_phi_row_split, 256-row granularity) with no collective, so rank r's whole work is
rf_phi_closed_form over rows [r0, r1) with the shared τ̂ and moments; the predicted R-GPU time is the max over ranks.
Each rank is timed --reps times back to back (CUDA events on the stream, median), ranks interleaved over --rounds.

  python scripts/phi_rank_emulation.py [--ranks 1,2,4,8] [--reps 20] [--rounds 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--ares", type=int, default=None, help="context option k5_ares (default: the library's)")
    ap.add_argument("--dyn", type=int, default=None, help="context option k5_dynamic (default: the library's)")
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    import synthetic
    cfg = synthetic.CONFIGS[4]
    n, p = cfg.n, cfg.p
    dev = torch.device("cuda:0")
    X = torch.from_numpy(synthetic.make_X(cfg)).to(torch.bfloat16).to(dev)
    Phi = torch.empty((n, n), dtype=torch.float32, device=dev)
    ws = torch.empty(rf.rf_phi_workspace_size(p, n, "bf16"), dtype=torch.uint8, device=dev)
    tau = rf.rf_estimate_tau(X)
    mom = rf.rf_moments(cfg.act, tau)
    tri = n * (n + 1) / 2.0
    ctx = rf.Context(0)
    if a.ares is not None:
        ctx.set_option("k5_ares", a.ares)
    if a.dyn is not None:
        ctx.set_option("k5_dynamic", a.dyn)

    def run(rb, re_):
        rf.rf_phi_closed_form(X, act=cfg.act, tau=tau, mom=mom, prec="bf16", out="upper", row_begin=rb, row_end=re_,
                              Phi=Phi, ws=ws, ctx=ctx)

    Rs = [int(v) for v in a.ranks.split(",")]
    times = {R: {r: [] for r in range(R)} for R in Rs}
    for _ in range(a.rounds):
        for R in Rs:
            for r in range(R):
                rb, re_ = rf.rf_phi_row_split(n, R, r)
                run(rb, re_)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.reps):
                    run(rb, re_)
                e1.record()
                e1.synchronize()
                times[R][r].append(e0.elapsed_time(e1) / a.reps)
    rows = []
    for R in Rs:
        per = [min(times[R][r]) for r in range(R)]
        rows.append({"R": R, "rank_ms": per, "step_ms": max(per), "entries_per_s": tri / (max(per) * 1e-3),
                     "rows": [rf.rf_phi_row_split(n, R, r) for r in range(R)]})
    base = rows[0]["step_ms"] if rows and rows[0]["R"] == 1 else None
    for row in rows:
        if base:
            row["speedup"] = base / row["step_ms"]
            row["efficiency"] = row["speedup"] / row["R"]
        print(json.dumps({k: v for k, v in row.items() if k != "rows"}), flush=True)
    print(json.dumps({"config": 4, "n": n, "p": p, "k5_ares": a.ares, "k5_dynamic": a.dyn, "rows": rows}))


if __name__ == "__main__":
    main()
