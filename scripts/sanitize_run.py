"""Drive every tensor-core kernel instantiation of the library once on small inputs, for the RF_DEBUG build
(device-side bounds checks on every store path, mbarrier-timeout and TMEM-allocation asserts; compute-sanitizer is
closed on this GPU pool, so these asserts stand in for memcheck).  Results are not checked here (the parity tests do
that); a failed check prints the offending index and traps.

  RF_B200_LIB=ab/librf_debug.so python scripts/sanitize_run.py [--big]
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(big: bool = "--big" in sys.argv):
    import numpy as np
    import torch
    import paper_2110_01899_b200 as rf
    import synthetic
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(0)

    def mk(n, p, dt):
        return torch.tensor(rng.standard_normal((n, p)) / math.sqrt(p), device=dev).to(dt)
    done = []
    # configs[0] shapes, every precision: K6 SIMT (fp64/fp32), K3/K4 pair kernels, 3×TF32 K-chunked K4, K5 (16 warps)
    cfg = synthetic.CONFIGS[0]
    for prec, dt in (("fp64", torch.float64), ("fp32", torch.float32), ("3xtf32", torch.float32),
                     ("tf32", torch.float32), ("bf16", torch.bfloat16)):
        X = torch.tensor(synthetic.make_X(cfg), device=dev).to(dt)
        W = torch.tensor(synthetic.make_W(cfg), device=dev).to(dt)
        rf.rf_gram(X, W, act="tanh", prec=prec, out="full")
        rf.rf_phi_closed_form(X, act="tanh", prec=prec, out="upper")
        if prec in ("bf16", "tf32", "3xtf32"):
            rf.rf_gram(X, W, act="tanh", prec=prec, out="packed_tri")
            rf.rf_phi_closed_form(X, act="tanh", prec=prec, out="packed_tri")
        done.append(f"configs[0] {prec}")
    # configs[1] slice (p = 784): K5 with 8 warps needs p > 512 → a p = 1024 slice as well
    X1 = torch.tensor(synthetic.make_X(1, n=1100, p=784), device=dev).float()
    W1 = torch.tensor(synthetic.make_W(1, m=700, p=784), device=dev).float()
    rf.rf_gram(X1, W1, act="erf", prec="3xtf32", out="upper")
    rf.rf_phi_closed_form(X1, act="erf", prec="3xtf32")
    rf.rf_phi_closed_form(mk(600, 1024, torch.bfloat16), act="tanh", prec="bf16")      # 8-warp K5
    rf.rf_phi_closed_form(X1.to(torch.bfloat16), act="relu", prec="bf16", form=2)      # general EQ1 / EQ2 epilogue
    done.append("configs[1] slice")
    # multicast + pair hybrids: K3 (≥ 32 row tiles) and K4 (≥ 64 row tiles), also the 8-CTA K4
    n = 16384 + 77 if big else 8448 + 77
    Xh, Wh = mk(n, 64, torch.bfloat16), mk(256, 64, torch.bfloat16)
    ctx = rf.Context(0)
    rf.rf_gram(Xh, Wh, act="tanh", prec="bf16", out="upper", ctx=ctx)
    if big:
        ctx.set_option("k4_cl8", 1)
        rf.rf_gram(Xh, Wh, act="tanh", prec="bf16", out="upper", ctx=ctx)
    done.append(f"hybrids n={n}")
    # G5 packed tiles: peers (world 1 and two emulated ranks with the phase hook), NCCL world 1
    for world in (1, 2):
        ctxs = [rf.Context(0) for _ in range(world)]
        for r, c in enumerate(ctxs):
            c.attach_peers(r, world, 1300)
        bases = [c.peer_base() for c in ctxs]
        for c in ctxs:
            c.connect_peers(bases)
        Xg, Wg = mk(1300, 96, torch.bfloat16), mk(512, 96, torch.bfloat16)
        for phase in ((1, 2) if world > 1 else (3,)):
            for r, c in enumerate(ctxs):
                c.set_option("g5_phases", phase)
                rf.rf_gram(Xg, Wg[r * 256:(r + 1) * 256].contiguous(), prec="bf16", out="packed_tiles", m_total=512,
                           ctx=c)
        torch.cuda.synchronize()
        for c in ctxs:
            c.destroy()
    done.append("G5 peers")
    # NEXT-1 (fp8 SYRK), NEXT-2 (K̃, centring), NEXT-4 (ridge)
    Xt = mk(700, 128, torch.bfloat16)
    Tt = torch.tensor(synthetic.make_T(0, 0.9, m=800, p=128), device=dev).to(torch.bfloat16)
    sm, sp = rf.rf_trf_thresholds_for("tanh", 1.0)
    rf.rf_gram_ter(Xt, Tt, 0.9, sm, sp, out="upper_centered")
    rf.rf_ktilde(Xt, torch.ones((700, 2), device=dev), np.eye(2), 0.1, 0.5, 0.2, prec="bf16")
    G = rf.rf_gram(Xt, mk(512, 128, torch.bfloat16), act="relu", prec="bf16", out="upper")
    rf.rf_ridge(G, 500, [0.1, 1.0], torch.ones((500, 1), dtype=torch.float64, device=dev))
    done.append("TRF, K̃, ridge")
    torch.cuda.synchronize()
    print("[sanitize_run] ok:", "; ".join(done), flush=True)


if __name__ == "__main__":
    main()
