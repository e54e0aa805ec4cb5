"""Timeline of bench.py's pipelined e2e leg (experiment): per-step compute and D2H intervals from CUDA events,
for the two step orders (G then Φ, Φ then G)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_01899_b200 as rf  # noqa: E402
import synthetic  # noqa: E402

dev = torch.device("cuda", 0)
cfg = synthetic.CONFIGS[3]
n, p, m = cfg.n, cfg.p, cfg.m
Xh = torch.from_numpy(synthetic.make_X(cfg)).bfloat16().pin_memory()
Wh = torch.from_numpy(synthetic.make_W(cfg)).bfloat16().pin_memory()
Xd, Wd = Xh.to(dev), Wh.to(dev)
ws_g = torch.empty(rf.rf_gram_workspace_size(p, n, m, "bf16"), dtype=torch.uint8, device=dev)
ws_p = torch.empty(rf.rf_phi_workspace_size(p, n, "bf16"), dtype=torch.uint8, device=dev)
E = rf.rf_packed_tri_elems(n)
bufs = [{"G": torch.empty(E, device=dev), "P": torch.empty(E, device=dev)} for _ in range(2)]
host = {"G": torch.empty(E, pin_memory=True), "P": torch.empty(E, pin_memory=True)}
st = torch.cuda.current_stream()
cs = torch.cuda.Stream()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    return e


def run(order, steps=6):
    done = [None, None]
    marks = []
    t0 = ev()
    t0.record(st)
    for k in range(steps):
        b = bufs[k & 1]
        if done[k & 1] is not None:
            st.wait_event(done[k & 1])
        Xd.copy_(Xh, non_blocking=True)
        Wd.copy_(Wh, non_blocking=True)
        rec = {}
        for what in order:
            a = ev(); a.record(st)
            if what == "G":
                rf.rf_gram(Xd, Wd, act=cfg.act, out="packed_tri", G=b["G"], ws=ws_g)
            else:
                rf.rf_phi_closed_form(Xd, act=cfg.act, out="packed_tri", Phi=b["P"], ws=ws_p)
            z = ev(); z.record(st)
            cs.wait_event(z)
            c0 = ev(); c0.record(cs)
            with torch.cuda.stream(cs):
                host[what].copy_(b[what], non_blocking=True)
            c1 = ev(); c1.record(cs)
            rec[what] = (a, z, c0, c1)
        d = torch.cuda.Event()
        d.record(cs)
        done[k & 1] = d
        marks.append(rec)
    st.wait_stream(cs)
    t1 = ev(); t1.record(st)
    torch.cuda.synchronize()
    tot = t0.elapsed_time(t1)
    print(f"order {''.join(order)}: {steps} steps {tot:.1f} ms = {tot / steps:.1f} ms/step")
    for k, rec in enumerate(marks):
        s = []
        for what, (a, z, c0, c1) in rec.items():
            s.append(f"{what}: comp {t0.elapsed_time(a):7.1f}-{t0.elapsed_time(z):7.1f}  d2h {t0.elapsed_time(c0):7.1f}-"
                     f"{t0.elapsed_time(c1):7.1f} ({E * 4 / (c0.elapsed_time(c1) * 1e-3) / 1e9:.1f} GB/s)")
        print(f"  step {k}: " + " | ".join(s))


for order in (["G", "P"], ["P", "G"], ["G", "P"], ["P", "G"]):
    run(order)
