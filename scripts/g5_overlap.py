"""Does the owner-side G5 sum hide under K4?  One B200, a world-1 peer context (the same kernels, streams and flags as a
rank of R, with every tile owned locally, so the sum reads one slice and writes recv: 2 × 8.6 GB at configs[3] — more
HBM traffic than an owner's sum at R = 8, 9.7 GB).  For K = m_local in --ms (m / R of configs[3]):
  dense     K3 + K4 into the dense upper triangle (no exchange)
  split     the collective call in its two halves, one after the other (phase 1: K3 + K4 packed + arrival flags;
            phase 2: the per-chunk sums + release flag) — the round-2 peer G5 without the pipeline
  piped     the collective call as the product runs it (phases 3: per-chunk flags on the comm stream, per-chunk sums
            on the reduce stream beside K4)
CUDA events on the caller's stream around each call, median of --reps after a warm-up.

  python scripts/g5_overlap.py [--ms 8192,65536] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="8192,65536")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    import synthetic
    cfg = synthetic.CONFIGS[3]
    n, p = cfg.n, cfg.p
    dev = torch.device("cuda:0")
    X = torch.from_numpy(synthetic.make_X(cfg)).to(torch.bfloat16).to(dev)
    W = torch.from_numpy(synthetic.make_W(cfg)).to(torch.bfloat16).to(dev)
    ctx = rf.Context(0)
    ctx.attach_peers(0, 1, n)
    ctxB = rf.Context(0)
    ctxB.attach_peers(0, 1, n)
    recv = torch.empty(len(rf.rf_tile_map(n, 1, 0)) * 65536, dtype=torch.float32, device=dev)
    G = torch.empty(n, n, dtype=torch.float32, device=dev)
    recvB = torch.empty_like(recv)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return sorted(ts)[len(ts) // 2]

    for m in [int(v) for v in a.ms.split(",")]:
        Wm = W[:m].contiguous()
        ws = torch.empty(rf.rf_workspace_size("gram", p, n, m, "bf16", "packed_tiles", ctx=ctx), dtype=torch.uint8,
                         device=dev)

        def coll(phase):
            ctx.set_option("g5_phases", phase)
            rf.rf_gram(X, Wm, act=cfg.act, prec="bf16", out="packed_tiles", m_total=cfg.m, G=recv, ws=ws, ctx=ctx)

        def split():
            coll(1)
            coll(2)

        t_dense = timed(lambda: rf.rf_gram(X, Wm, act=cfg.act, prec="bf16", out="upper", G=G, ws=ws, ctx=ctx))
        t_split = timed(split)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        coll(1)
        e[1].record()
        coll(2)
        e[2].record()
        e[2].synchronize()
        t_piped = timed(lambda: coll(3))
        torch.cuda.synchronize()
        rf.rf_profile_read()
        rf.rf_profile_enable(True)
        coll(3)
        torch.cuda.synchronize()
        rf.rf_profile_enable(False)
        tl = [(nm, round(t0, 2), round(ms, 3)) for nm, t0, ms in rf.rf_profile_timeline()]
        # co-residency check with the packed K4 (129 registers: room for a sum CTA beside it): a second world-1
        # context B runs phase 1 (its tiles in its staging buffer), then context A's phase 1 (K3 + packed K4) on the
        # current stream and B's per-chunk sums (phase 2, flags already up) on a side stream right behind it; the sums
        # ending long before K4 means they ran on the SMs beside it
        ctxB.set_option("g5_phases", 1)
        rf.rf_gram(X, Wm, act=cfg.act, prec="bf16", out="packed_tiles", m_total=cfg.m, G=recvB, ws=ws, ctx=ctxB)
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        c0, c1, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        c0.record()
        coll(1)
        c1.record()
        side.wait_event(c0)
        ctxB.set_option("g5_phases", 2)
        rf.rf_gram(X, Wm, act=cfg.act, prec="bf16", out="packed_tiles", m_total=cfg.m, G=recvB, ws=ws, ctx=ctxB,
                   stream=side)
        c2.record(side)
        torch.cuda.synchronize()
        coll(2)
        ctx.set_option("g5_phases", 3)
        conc = {"k3_k4_packed_end_ms": c0.elapsed_time(c1), "sums_end_ms": c0.elapsed_time(c2)}
        print(json.dumps({"m_local": m, "dense_ms": t_dense, "split_ms": t_split, "split_phase1_ms": e[0].elapsed_time(e[1]),
                          "split_phase2_ms": e[1].elapsed_time(e[2]), "piped_ms": t_piped,
                          "piped_exposed_vs_dense_ms": t_piped - t_dense, "concurrent": conc, "piped_timeline": tl, "sum_bytes_gb": 2 * recv.numel() * 4 / 1e9}),
              flush=True)
        del ws
    ctx.destroy()


if __name__ == "__main__":
    main()
