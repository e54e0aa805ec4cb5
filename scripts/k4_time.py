"""K3/K4 device times at BASELINE.json configs[3] (p = 1024, n = m = 65536, bf16, sigmoid − ½): CUDA events recorded by
the library around each launch (the hybrids' two kernels separately as *_mc / *_tail), median over reps, for the
context options given (A/B runs interleave them).

  python scripts/k4_time.py [--reps 3] [--opts k4_dynamic=1 k4_dynamic=0 ...]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--opts", nargs="*", default=["k4_dynamic=1", "k4_dynamic=0"])
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    import synthetic
    cfg = synthetic.CONFIGS[3]
    dev = torch.device("cuda:0")
    X = torch.from_numpy(synthetic.make_X(cfg)).to(torch.bfloat16).to(dev)
    W = torch.from_numpy(synthetic.make_W(cfg)).to(torch.bfloat16).to(dev)
    G = torch.empty(cfg.n, cfg.n, device=dev)
    ws = torch.empty(rf.rf_gram_workspace_size(cfg.p, cfg.n, cfg.m, "bf16"), dtype=torch.uint8, device=dev)
    ctx = rf.Context(0)
    fl4 = cfg.m * cfg.n * (cfg.n + 1.0)
    for _ in range(a.rounds):
        for o in a.opts:
            k, v = o.split("=")
            ctx.set_option(k, int(v))
            rf.rf_gram(X, W, act=cfg.act, prec="bf16", G=G, ws=ws, ctx=ctx)
            torch.cuda.synchronize()
            rf.rf_profile_read()
            rf.rf_profile_enable(True)
            for _ in range(a.reps):
                rf.rf_gram(X, W, act=cfg.act, prec="bf16", G=G, ws=ws, ctx=ctx)
            torch.cuda.synchronize()
            rf.rf_profile_enable(False)
            rec = {}
            for nm, ms in rf.rf_profile_read():
                rec.setdefault(nm, []).append(ms)
            med = {nm: sorted(v)[len(v) // 2] for nm, v in rec.items()}
            print(json.dumps({"opt": o, "K4_ms": med.get("K4_syrk"), "K4_tflops": fl4 / med["K4_syrk"] / 1e9,
                              "K4_mc_ms": med.get("K4_syrk_mc"), "K4_tail_ms": med.get("K4_syrk_tail"),
                              "K3_ms": med.get("K3_gemm_sigma")}), flush=True)


if __name__ == "__main__":
    main()
