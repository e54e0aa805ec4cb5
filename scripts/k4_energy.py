"""Experiment: K3/K4 device time, SM clock and board power on configs[3]-shaped inputs, swept over the K4 soft
lockstep window (context option lock_w) and over operand data (random vs all-zero Σ, to see how much of the
power-capped clock is data-dependent).  Not part of the product path; run under gpurun.

  python scripts/k4_energy.py [--lockw 0,24] [--zero] [--reps 3]
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--m", type=int, default=65536)
    ap.add_argument("--p", type=int, default=1024)
    ap.add_argument("--pad-g", action="store_true")
    ap.add_argument("--lockw", default="24")
    ap.add_argument("--zero", action="store_true", help="also time with W = 0 (Σ = σ(0) = 0)")
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    X = (torch.randn(a.n, a.p, device=dev, generator=g) / a.p ** 0.5).to(torch.bfloat16)
    W = torch.randn(a.m, a.p, device=dev, generator=g).to(torch.bfloat16)
    ldg = a.n + 32 if a.pad_g else a.n          # odd number of 128-B lines per row (see api.cu odd_line_ld)
    G = torch.empty(a.n, ldg, device=dev)[:, :a.n]
    ws = torch.empty(rf.rf_gram_workspace_size(a.p, a.n, a.m, "bf16"), dtype=torch.uint8, device=dev)
    rf.rf_profile_enable(True)
    ctx = rf.Context(0)
    cases = [("rand", W, lw) for lw in a.lockw.split(",")]
    if a.zero:
        cases.append(("zero", torch.zeros_like(W), a.lockw.split(",")[-1]))
    for tag, Wc, lw in cases:
        ctx.set_option("lock_w", int(lw))
        rf.rf_gram(X, Wc, act="sigmoid_half", prec="bf16", G=G, ws=ws, ctx=ctx)
        torch.cuda.synchronize()
        rf.rf_profile_read()
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                "-lms", "100"], stdout=subprocess.PIPE, text=True)
        time.sleep(0.3)
        for _ in range(a.reps):
            rf.rf_gram(X, Wc, act="sigmoid_half", prec="bf16", G=G, ws=ws, ctx=ctx)
        torch.cuda.synchronize()
        smi.terminate()
        out = smi.communicate()[0]
        rec = rf.rf_profile_read()
        k3 = [ms for nm, ms in rec if nm.startswith("K3")]
        k4 = [ms for nm, ms in rec if nm.startswith("K4")]
        vals = [l.split(",") for l in out.strip().splitlines() if l.strip()]
        clk = sorted(float(v[0]) for v in vals if len(v) == 2)
        pw = sorted(float(v[1]) for v in vals if len(v) == 2)
        busy = [c for c in clk]
        med = lambda x: x[len(x) // 2] if x else float("nan")
        fl4 = a.m * a.n * (a.n + 1)
        fl3 = 2.0 * a.m * a.n * a.p
        print(f"[{tag} lockw={lw}] K3 {med(sorted(k3)):.2f} ms ({fl3 / med(sorted(k3)) / 1e9:.0f} TF/s)  "
              f"K4 {med(sorted(k4)):.2f} ms ({fl4 / med(sorted(k4)) / 1e9:.0f} TF/s)  "
              f"sm_mhz med {med(busy):.0f} (min {busy[0] if busy else 0:.0f})  power med {med(pw):.0f} W max "
              f"{pw[-1] if pw else 0:.0f} W  samples {len(clk)}", flush=True)


if __name__ == "__main__":
    main()
