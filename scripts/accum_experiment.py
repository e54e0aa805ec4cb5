"""Measure the tensor-pipe accumulation error of the tcgen05 mainloop vs K and vs the K-chunk size.

SYRK-like inputs: A = B = rows of σ-like values in (−1, 1) (tf32/bf16 representable, so products are
exact and every error comes from accumulation).  Prints mean signed relative error on the diagonal
(all-positive sums: exposes a rounding bias) and relative Frobenius error over the whole matrix.
Usage (GPU): python scripts/accum_experiment.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_01899_b200 as rf  # noqa: E402


def run(prec, K, kchunk, n=512, seed=0):
    rng = np.random.default_rng(seed)
    S = np.tanh(rng.standard_normal((n, K)))
    if prec == "bf16":
        St = torch.tensor(S, device="cuda").to(torch.bfloat16)
    else:
        St = torch.tensor(S, device="cuda").float()
        if prec == "tf32":   # make the operand exactly tf32-representable
            St = (St.view(torch.int32) & ~0x1FFF).view(torch.float32)
    S64 = St.double().cpu().numpy()
    C = rf.rf_debug_gemm_nt(St, St, prec=prec, kchunk=kchunk).double().cpu().numpy()
    ref = S64 @ S64.T
    d = np.arange(n)
    bias = float(np.mean((C[d, d] - ref[d, d]) / ref[d, d]))
    fro = float(np.linalg.norm(C - ref) / np.linalg.norm(ref))
    return bias, fro


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for prec in ("tf32", "bf16", "3xtf32"):
        for K in (1024, 8192, 32768):
            for kchunk in (0, 64, 16, 8, 4, 2, 1):
                kb = 64 if prec == "bf16" else 32
                if kchunk and kchunk * kb >= K:
                    continue
                b, f = run(prec, K, kchunk)
                print(f"{prec:7s} K={K:6d} kchunk={kchunk:3d} (Kc={kchunk * kb if kchunk else K:6d}): "
                      f"diag mean rel err {b:+.3e}  rel-Frobenius {f:.3e}", flush=True)
