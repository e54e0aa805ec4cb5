"""Experiment: K5 (fused XᵀX + EQ1 epilogue) device time on configs-shaped bf16 inputs, with the achieved
tensor TFLOP/s (p·n(n+1) algorithmic) and HBM GB/s (fp32 upper triangle written + X read).  Not part of
the product path; run under gpurun.

  python scripts/k5_bench.py [--n 131072 --p 512] [--reps 3] [--prec bf16]
"""
import argparse
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--p", type=int, default=512)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--prec", default="bf16")
    ap.add_argument("--act", default="tanh")
    ap.add_argument("--pad", type=int, default=0, help="extra fp32 elements per row of Φ (leading dimension n + pad)")
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    X = torch.randn(a.n, a.p, device=dev, generator=g)
    X = X / X.norm(dim=1, keepdim=True) * (0.5 + torch.rand(a.n, 1, device=dev, generator=g))
    X = X.to(torch.bfloat16 if a.prec == "bf16" else torch.float32)
    ldp = a.n + a.pad
    Phi = torch.empty(a.n, ldp, device=dev)[:, :a.n]
    ws = torch.empty(rf.rf_phi_workspace_size(a.p, a.n, a.prec), dtype=torch.uint8, device=dev)
    tau = rf.rf_estimate_tau(X)
    mom = rf.rf_moments(a.act, tau)
    rf.rf_profile_enable(True)
    rf.rf_phi_closed_form(X, act=a.act, tau=tau, mom=mom, prec=a.prec, Phi=Phi, ws=ws)
    torch.cuda.synchronize()
    rf.rf_profile_read()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    for _ in range(a.reps):
        rf.rf_phi_closed_form(X, act=a.act, tau=tau, mom=mom, prec=a.prec, Phi=Phi, ws=ws)
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0]
    rec = rf.rf_profile_read()
    k5 = sorted(ms for nm, ms in rec if nm.startswith("K5"))
    med = k5[len(k5) // 2]
    vals = [l.split(",") for l in out.strip().splitlines() if l.strip()]
    clk = sorted(float(v[0]) for v in vals if len(v) == 2)
    tri = a.n * (a.n + 1) / 2
    fl = a.p * a.n * (a.n + 1.0)
    by = 4 * tri + X.numel() * X.element_size()
    print(f"[K5 n={a.n} p={a.p} {a.prec} {a.act} pad={a.pad}] {med:.3f} ms  {fl / med / 1e9:.0f} TF/s  {by / med / 1e6:.0f} GB/s  "
          f"{tri / med / 1e9:.1f} G entries/s  sm_mhz med {clk[len(clk) // 2] if clk else 0:.0f}  all {[round(x, 3) for x in k5]}",
          flush=True)


if __name__ == "__main__":
    main()
