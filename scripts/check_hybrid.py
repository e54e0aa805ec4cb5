"""Check: the hybrid K4 launch (4-CTA multicast clusters + pair clusters on a side stream) equals the pair-only K4
bit for bit, for the bf16 Gram and the fp8 ternary Gram."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01899_b200 as rf
for n, p, m in [(16384, 128, 1024), (20000, 64, 2048)]:
    g = torch.Generator(device="cuda").manual_seed(n)
    X = (torch.randn(n, p, device="cuda", generator=g) / p ** 0.5).to(torch.bfloat16)
    W = torch.randn(m, p, device="cuda", generator=g).to(torch.bfloat16)
    T = torch.randint(-1, 2, (m, p), device="cuda", generator=g).to(torch.bfloat16)
    out = {}
    for h in ("0", "1"):
        os.environ["RF_K4_HYBRID"] = h
        Gg = rf.rf_gram(X, W, act="tanh", prec="bf16", out="upper")
        Gt = rf.rf_gram_ter(X, T, 0.5, -0.4, 0.4, out="upper")
        torch.cuda.synchronize()
        out[h] = (Gg.triu(), Gt.triu())
    print(n, "gram", "bit-exact" if torch.equal(out["0"][0], out["1"][0]) else "DIFF",
          "ter", "bit-exact" if torch.equal(out["0"][1], out["1"][1]) else "DIFF", flush=True)
