"""Per-rank Φ time at configs[4], R = 8 row blocks, rank order forward / reversed, and with an odd-line leading dimension
(timing probe for DESIGN.md §9)."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2110_01899_b200 as rf, synthetic
cfg = synthetic.CONFIGS[4]; n, p = cfg.n, cfg.p
X = torch.from_numpy(synthetic.make_X(cfg)).to(torch.bfloat16).cuda()
if "--roll" in sys.argv:   # move the data: row i gets sample (i + 40000) mod n (is the slow rank about data or position?)
    X = torch.roll(X, shifts=-40000, dims=0).contiguous()
PhiA = torch.empty((n, n), device="cuda")
PhiB = torch.empty((n, n + 32), device="cuda")[:, :n]   # odd number of 128-B lines per row
ws = torch.empty(rf.rf_phi_workspace_size(p, n, "bf16"), dtype=torch.uint8, device="cuda")
tau = rf.rf_estimate_tau(X); mom = rf.rf_moments(cfg.act, tau)
def t(r, Phi, reps=20):
    rb, re_ = rf.rf_phi_row_split(n, 8, r)
    f = lambda: rf.rf_phi_closed_form(X, act=cfg.act, tau=tau, mom=mom, prec="bf16", row_begin=rb, row_end=re_, Phi=Phi, ws=ws)
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); b.synchronize()
    return round(a.elapsed_time(b) / reps, 3)
for rnd in range(2):
    print("A fwd", [t(r, PhiA) for r in range(8)])
    print("A rev", [t(r, PhiA) for r in reversed(range(8))][::-1])
    print("B(ld+32) fwd", [t(r, PhiB) for r in range(8)])
print("splits", [rf.rf_phi_row_split(n, 8, r) for r in range(8)])
