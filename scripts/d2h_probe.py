"""Host-link probe for the e2e leg: D2H / H2D bandwidth of large pinned copies, one or several streams, alone and
while a K4-sized SYRK runs (experiment, not product code)."""
import sys
import time

import torch

sys.path.insert(0, ".")
dev = torch.device("cuda", 0)
GB = 1 << 30
nbytes = 8 * GB
src = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
dst = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
print("pinned alloc ok", flush=True)


def run(nstreams, chunk_mb, direction="d2h"):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    ce = chunk_mb * (1 << 20) // 4
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, off in enumerate(range(0, src.numel(), ce)):
        with torch.cuda.stream(streams[i % nstreams]):
            if direction == "d2h":
                dst[off:off + ce].copy_(src[off:off + ce], non_blocking=True)
            else:
                src[off:off + ce].copy_(dst[off:off + ce], non_blocking=True)
    torch.cuda.synchronize()
    return nbytes / (time.perf_counter() - t0) / 1e9


for d in ("d2h", "h2d"):
    for ns, cm in [(1, 8192), (1, 256), (2, 256), (4, 256), (4, 64), (8, 32)]:
        run(ns, cm, d)
        print(f"{d} streams={ns} chunk={cm}MB: {run(ns, cm, d):.1f} GB/s", flush=True)

# D2H while the SYRK of configs[3] runs
import paper_2110_01899_b200 as rf
import synthetic
cfg = synthetic.CONFIGS[3]
X = torch.from_numpy(synthetic.make_X(cfg)).bfloat16().to(dev)
W = torch.from_numpy(synthetic.make_W(cfg)).bfloat16().to(dev)
G = torch.empty(rf.rf_packed_tri_elems(cfg.n), device=dev)
ws = torch.empty(rf.rf_gram_workspace_size(cfg.p, cfg.n, cfg.m, "bf16"), dtype=torch.uint8, device=dev)
rf.rf_gram(X, W, act=cfg.act, out="packed_tri", G=G, ws=ws)
torch.cuda.synchronize()
cs = torch.cuda.Stream()
t0 = time.perf_counter()
rf.rf_gram(X, W, act=cfg.act, out="packed_tri", G=G, ws=ws)
with torch.cuda.stream(cs):
    dst.copy_(src, non_blocking=True)
e = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
print(f"gram ∥ 8 GiB D2H: {time.perf_counter() - t0:.3f} s total", flush=True)
t0 = time.perf_counter()
rf.rf_gram(X, W, act=cfg.act, out="packed_tri", G=G, ws=ws)
torch.cuda.synchronize()
print(f"gram alone: {time.perf_counter() - t0:.3f} s", flush=True)
t0 = time.perf_counter()
dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
print(f"8 GiB D2H alone: {time.perf_counter() - t0:.3f} s", flush=True)

# D2H rate measured on the copy stream itself (events), in 256-MB pieces, alone and under the SYRK
def d2h_events(with_gram):
    ce = (256 << 20) // 4
    torch.cuda.synchronize()
    if with_gram:
        rf.rf_gram(X, W, act=cfg.act, out="packed_tri", G=G, ws=ws)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        a.record(cs)
        for off in range(0, src.numel(), ce):
            dst[off:off + ce].copy_(src[off:off + ce], non_blocking=True)
        b.record(cs)
    torch.cuda.synchronize()
    return nbytes / (a.elapsed_time(b) * 1e-3) / 1e9


for rep in range(2):
    print(f"D2H 256-MB pieces, alone: {d2h_events(False):.1f} GB/s; under K3+K4: {d2h_events(True):.1f} GB/s", flush=True)
