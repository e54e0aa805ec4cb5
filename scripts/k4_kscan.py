"""K4 device time against the SYRK depth K = m at n = 65536 (p = 1024, bf16, sigmoid − ½): separates the per-tile fixed
cost (accumulator hand-off + epilogue drain, paid once per output tile) from the K-proportional MMA time.  At R GPUs a
rank's K4 runs with K = m/R, so the fixed cost is what the strong-scaling curve loses.

  python scripts/k4_kscan.py [--ms 8192,16384,65536] [--reps 3] [--opts k4_epi16=0 k4_epi16=1] [--packed]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="8192,16384,65536")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--opts", nargs="*", default=[""])
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    import synthetic
    cfg = synthetic.CONFIGS[3]
    dev = torch.device("cuda:0")
    X = torch.from_numpy(synthetic.make_X(cfg)).to(torch.bfloat16).to(dev)
    W = torch.from_numpy(synthetic.make_W(cfg)).to(torch.bfloat16).to(dev)
    G = torch.empty(cfg.n, cfg.n, device=dev)
    ctx = rf.Context(0)
    for _ in range(a.rounds):
        for m in [int(v) for v in a.ms.split(",")]:
            Wm = W[:m].contiguous()
            ws = torch.empty(rf.rf_gram_workspace_size(cfg.p, cfg.n, m, "bf16"), dtype=torch.uint8, device=dev)
            fl4 = m * cfg.n * (cfg.n + 1.0)
            for o in a.opts:
                if o:
                    k, v = o.split("=")
                    ctx.set_option(k, int(v))
                rf.rf_gram(X, Wm, act=cfg.act, prec="bf16", G=G, ws=ws, ctx=ctx)
                torch.cuda.synchronize()
                rf.rf_profile_read()
                rf.rf_profile_enable(True)
                for _ in range(a.reps):
                    rf.rf_gram(X, Wm, act=cfg.act, prec="bf16", G=G, ws=ws, ctx=ctx)
                torch.cuda.synchronize()
                rf.rf_profile_enable(False)
                rec = {}
                for nm, ms in rf.rf_profile_read():
                    rec.setdefault(nm, []).append(ms)
                med = {nm: sorted(v)[len(v) // 2] for nm, v in rec.items()}
                print(json.dumps({"m": m, "opt": o, "K4_ms": med.get("K4_syrk"),
                                  "K4_tflops": fl4 / med["K4_syrk"] / 1e9, "K4_mc_ms": med.get("K4_syrk_mc"),
                                  "K4_tail_ms": med.get("K4_syrk_tail"), "K3_ms": med.get("K3_gemm_sigma")}),
                      flush=True)
            del ws


if __name__ == "__main__":
    main()
