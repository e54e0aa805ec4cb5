"""Probe: HBM write-only bandwidth on this B200 (fill of a large fp32 buffer) vs copy (read+write)."""
import torch
x = torch.empty(8 * 1024**3 // 4, dtype=torch.float32, device="cuda")   # 8 GiB
y = torch.empty_like(x)
for name, fn, by in [("fill", lambda: x.fill_(1.5), x.numel() * 4), ("zero", lambda: x.zero_(), x.numel() * 4),
                     ("copy", lambda: y.copy_(x), 2 * x.numel() * 4)]:
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"{name}: {by / ms / 1e6:.0f} GB/s ({ms:.2f} ms)")
