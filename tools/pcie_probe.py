"""Pinned host<->device copy rate for the e2e leg's buffer size (8 MB FP64 vector)."""
import torch

n = 1 << 20
h = torch.randn(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(50):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"{name}: {ms*1e3:.1f} us per 8 MB = {8 * 2**20 / ms / 1e6:.1f} GB/s")
