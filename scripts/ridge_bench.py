"""NEXT-4 timing breakdown (experiment): rf_ridge device time per kernel family and wall time, at the paper's
ridge size (n_train = 1024, 7 γ) and a large single-γ factorisation (n = 16384)."""
import os
import sys
import time
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_01899_b200 as rf  # noqa: E402
import synthetic  # noqa: E402

dev = torch.device("cuda:0")
for n_tr, n_te, gam in [(1024, 512, [1e-2, 1e-1, 1.0, 10.0, 1e2, 1e3, 1e4]), (16384, 0, [1.0])]:
    X, y = synthetic.make_ridge_gmm(n_tr, n_te, 512)
    Xd = torch.from_numpy(X).bfloat16().to(dev)
    Wd = torch.from_numpy(synthetic.make_W(1, m=4096, p=512)).bfloat16().to(dev)
    G = rf.rf_gram(Xd, Wd, act="relu", prec="bf16", out="upper")
    Y = torch.from_numpy(y[:n_tr]).to(dev)
    ws = torch.empty(rf.rf_ridge_workspace_size(n_tr), dtype=torch.uint8, device=dev)
    rf.rf_ridge(G, n_tr, gam, Y, n_test=n_te)
    torch.cuda.synchronize()
    rf.rf_profile_read()
    rf.rf_profile_enable(True)
    t0 = time.perf_counter()
    rf.rf_ridge(G, n_tr, gam, Y, n_test=n_te)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    rf.rf_profile_enable(False)
    agg = defaultdict(lambda: [0, 0.0])
    for nm, ms in rf.rf_profile_read(100000):
        agg[nm][0] += 1
        agg[nm][1] += ms
    dev_ms = sum(v[1] for v in agg.values())
    print(f"[ridge n={n_tr}+{n_te} γ×{len(gam)}] wall {wall:.2f} ms, device sum {dev_ms:.2f} ms, launches "
          f"{sum(v[0] for v in agg.values())}: " + ", ".join(f"{k} {v[0]}×/{v[1]:.2f} ms" for k, v in sorted(agg.items())),
          flush=True)
