"""Can other kernels run on the SMs beside K4?  One B200: K4 (dense K3 + K4 at configs[3] with m = --m) on the current
stream; on a second stream, --copies device copies of --mb MB each (torch's elementwise copy kernel), launched right
after.  Prints the copies' total time alone, K4 alone, and both together with each copy's finish time relative to the
start of K4: copies that finish long before K4 ends ran on the SMs beside it.

  python scripts/coresidency_probe.py [--m 65536] [--copies 16] [--mb 512]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=65536)
    ap.add_argument("--copies", type=int, default=16)
    ap.add_argument("--mb", type=int, default=512)
    a = ap.parse_args()
    import torch
    import paper_2110_01899_b200 as rf
    import synthetic
    cfg = synthetic.CONFIGS[3]
    dev = torch.device("cuda:0")
    X = torch.from_numpy(synthetic.make_X(cfg)).to(torch.bfloat16).to(dev)
    W = torch.from_numpy(synthetic.make_W(cfg))[: a.m].to(torch.bfloat16).to(dev)
    G = torch.empty(cfg.n, cfg.n, device=dev)
    src = [torch.ones(a.mb << 18, device=dev) for _ in range(a.copies)]
    dst = [torch.empty_like(x) for x in src]
    side = torch.cuda.Stream()
    ctx = rf.Context(0)

    def k4():
        rf.rf_gram(X, W, act=cfg.act, prec="bf16", G=G, ctx=ctx)

    def copies(stream, marks):
        with torch.cuda.stream(stream):
            for d, s_ in zip(dst, src):
                d.copy_(s_)
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks.append(e)

    for _ in range(2):
        k4()
        copies(torch.cuda.current_stream(), [])
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    copies(torch.cuda.current_stream(), (m0 := []))
    torch.cuda.synchronize()
    alone_copies = t0.elapsed_time(m0[-1])
    t0.record()
    k4()
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    torch.cuda.synchronize()
    alone_k4 = t0.elapsed_time(t1)
    t0.record()
    k4()
    t1.record()
    side.wait_event(t0)
    copies(side, (m1 := []))
    torch.cuda.synchronize()
    print(json.dumps({"m": a.m, "copies_alone_ms": alone_copies, "k4_alone_ms": alone_k4,
                      "k4_with_copies_ms": t0.elapsed_time(t1),
                      "copy_finish_ms_from_k4_start": [round(t0.elapsed_time(e), 2) for e in m1]}))


if __name__ == "__main__":
    main()
