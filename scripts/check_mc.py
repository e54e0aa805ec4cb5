"""Check: K4 with 4-CTA clusters + B multicast (RF_K4_MC=1) equals the pair-cluster K4 bit for bit."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2110_01899_b200 as rf
for n, p, m in [(600, 64, 384), (1300, 128, 1000), (2048, 256, 4096), (4100, 128, 3000)]:
    g = torch.Generator(device="cuda").manual_seed(n)
    X = (torch.randn(n, p, device="cuda", generator=g) / p ** 0.5).to(torch.bfloat16)
    W = torch.randn(m, p, device="cuda", generator=g).to(torch.bfloat16)
    os.environ["RF_K4_MC"] = "0"
    G0 = rf.rf_gram(X, W, act="tanh", prec="bf16", out="upper")
    os.environ["RF_K4_MC"] = "1"
    G1 = rf.rf_gram(X, W, act="tanh", prec="bf16", out="upper")
    torch.cuda.synchronize()
    iu = torch.triu_indices(n, n, device="cuda")
    a, b = G0[iu[0], iu[1]], G1[iu[0], iu[1]]
    print(n, p, m, "bit-exact" if torch.equal(a, b) else f"DIFF max {float((a - b).abs().max()):.3e}", flush=True)
