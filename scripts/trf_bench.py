"""Timing of the TRF path (NEXT-1) on configs[3] sizes: K3^ter (bf16 X·Tᵀ + σ^ter → fp8) and K4^ter (fp8
SYRK) device times, clocks.  Not part of the product path; run under gpurun.

  python scripts/trf_bench.py [--eps 0.9] [--reps 3]
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
    ap.add_argument("--eps", type=float, default=0.9)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--m", type=int, default=65536)
    ap.add_argument("--p", type=int, default=1024)
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    X = (torch.randn(a.n, a.p, device=dev, generator=g) / a.p ** 0.5).to(torch.bfloat16)
    u = torch.rand(a.m, a.p, device=dev, generator=g)
    T = torch.where(u < a.eps, 0.0, torch.where(u < a.eps + (1 - a.eps) / 2, -1.0, 1.0)).to(torch.bfloat16)
    tau = rf.rf_estimate_tau(X)
    sm, sp = rf.rf_trf_thresholds_for("sigmoid_half", tau)
    G = torch.empty(a.n, a.n, device=dev)
    ws = torch.empty(rf.rf_gram_ter_workspace_size(a.p, a.n, a.m), dtype=torch.uint8, device=dev)
    rf.rf_profile_enable(True)
    rf.rf_gram_ter(X, T, a.eps, sm, sp, G=G, ws=ws)
    torch.cuda.synchronize()
    rf.rf_profile_read()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    for _ in range(a.reps):
        rf.rf_gram_ter(X, T, a.eps, sm, sp, G=G, ws=ws)
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0]
    rec = rf.rf_profile_read()
    med = lambda x: sorted(x)[len(x) // 2]
    k3 = med([ms for nm, ms in rec if nm.startswith("K3")])
    k4 = med([ms for nm, ms in rec if nm.startswith("K4")])
    clk = sorted(float(l.split(",")[0]) for l in out.strip().splitlines() if "," in l)
    fl3 = 2.0 * a.m * a.n * a.p
    fl4 = a.m * a.n * (a.n + 1.0)
    print(f"[TRF eps={a.eps} n={a.n} m={a.m} p={a.p} s=({sm:.4f},{sp:.4f})] K3^ter {k3:.2f} ms "
          f"({fl3 / k3 / 1e9:.0f} TF/s bf16)  K4^ter {k4:.2f} ms ({fl4 / k4 / 1e9:.0f} TF/s fp8)  "
          f"step {(fl3 + fl4) / (k3 + k4) / 1e9:.0f} TF/s  sm_mhz med {clk[len(clk) // 2] if clk else 0:.0f}", flush=True)


if __name__ == "__main__":
    main()
