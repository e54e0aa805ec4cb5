"""K5 (fused XᵀX + EQ1 epilogue) device time at BASELINE.json configs[4] (n = 131072, p = 512, bf16 X, tanh, fp32
upper triangle): CUDA events recorded by the library around each launch, with the algorithmic HBM GB/s
(4 B per upper-triangle entry + X) and TFLOP/s (p·n(n+1)).  RF_B200_LIB selects another build for A/B runs.

  python scripts/k5_time.py [--n 131072 --p 512 --reps 5 --wide -1 --out upper]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--p", type=int, default=512)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--wide", type=int, default=-1)
    ap.add_argument("--out", default="upper")
    ap.add_argument("--act", default="tanh")
    ap.add_argument("--ares", type=int, default=None, help="context option k5_ares (A-panel residency; default: the "
                    "library's)")
    ap.add_argument("--prec", default="bf16", choices=["bf16", "tf32"])
    ap.add_argument("--clocks", action="store_true", help="sample SM clock / power / throttle reasons (nvidia-smi) "
                    "over the timed launches (use --reps ≥ 200 so the 200-ms sampler sees them)")
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    import synthetic
    dev = torch.device("cuda:0")
    cfg = synthetic.CONFIGS[4]
    X = torch.from_numpy(synthetic.make_X(cfg, n=a.n, p=a.p)).to(torch.bfloat16 if a.prec == "bf16" else torch.float32)
    X = X.to(dev)
    ctx = rf.Context(0) if hasattr(rf, "Context") else None
    if ctx is not None:
        ctx.set_option("k5_wide", a.wide)
        if a.ares is not None:
            ctx.set_option("k5_ares", a.ares)
    Phi = (torch.empty(rf.rf_packed_tri_elems(a.n), device=dev) if a.out == "packed_tri"
           else torch.empty(a.n, a.n, device=dev))
    ws = torch.empty(rf.rf_phi_workspace_size(a.p, a.n, a.prec), dtype=torch.uint8, device=dev)
    tau = rf.rf_estimate_tau(X)
    mom = rf.rf_moments(a.act, tau)
    kw = {"ctx": ctx} if ctx is not None else {}
    for _ in range(2):
        rf.rf_phi_closed_form(X, act=a.act, tau=tau, mom=mom, prec=a.prec, out=a.out, Phi=Phi, ws=ws, **kw)
    torch.cuda.synchronize()
    rf.rf_profile_read()
    rf.rf_profile_enable(True)
    sampler = None
    if a.clocks:
        import bench
        sampler = bench.ClockSampler([0])
    for _ in range(a.reps):
        rf.rf_phi_closed_form(X, act=a.act, tau=tau, mom=mom, prec=a.prec, out=a.out, Phi=Phi, ws=ws, **kw)
    torch.cuda.synchronize()
    clk = sampler.stop() if sampler is not None else None
    ks = [t for nm, t in rf.rf_profile_read() if nm.startswith("K5")]
    ks.sort()
    med = ks[len(ks) // 2]
    tri = a.n * (a.n + 1) / 2.0
    by = 4.0 * tri + 2.0 * a.n * a.p
    print(json.dumps({"lib": os.environ.get("RF_B200_LIB", "in-tree"), "n": a.n, "p": a.p, "wide": a.wide, "ares": a.ares, "prec": a.prec,
                      "out": a.out, "k5_ms_median": med, "k5_ms_min": ks[0], "k5_ms_all": ks if len(ks) <= 10 else None,
                      "hbm_gbs": by / (med * 1e-3) / 1e9, "tflops": a.p * a.n * (a.n + 1.0) / (med * 1e-3) / 1e12,
                      "clocks": clk}))


if __name__ == "__main__":
    main()
