"""HBM write-only ceiling on this GPU: fill_ / zero_ of a 3.2 GB fp32 buffer (CUDA events).

The decode kernel's roofline denominator is the measured copy bandwidth
(MEASURED_PEAKS.json); this reports what a pure streaming write reaches, for context.
"""
import torch

n = 800 * 1024 * 1024  # 3.36 GB of fp32, about one decode level
x = torch.empty(n, dtype=torch.float32, device="cuda")
y = torch.empty(n, dtype=torch.float32, device="cuda")
for name, fn in (("fill_", lambda: x.fill_(1.0)), ("zero_", lambda: x.zero_()), ("copy_", lambda: y.copy_(x))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    nbytes = x.numel() * 4 * (2 if name == "copy_" else 1)
    print(f"{name}: {nbytes / best / 1e6:.0f} GB/s ({best:.3f} ms for {nbytes / 1e9:.2f} GB)")
