"""HBM write-only and copy bandwidth (fill / copy of 411 MB, VGG conv1_x output size)."""
import torch

n = 32 * 224 * 224 * 64
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
for name, fn in (("fill (write only)", lambda: a.fill_(1.0)), ("copy (read+write)", lambda: b.copy_(a))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    moved = 4 * n * (1 if "fill" in name else 2)
    print(f"{name}: {ms * 1e3:.1f} us for {moved / 1e6:.0f} MB -> {moved / ms / 1e6:.0f} GB/s")
