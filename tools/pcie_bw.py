"""Host<->device copy bandwidth from page-locked memory (the e2e bound)."""
import torch

n = 256 << 20
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s2 = torch.cuda.Stream()
h2 = torch.empty_like(h).pin_memory()
d2 = torch.empty_like(d)
for name in ("h2d", "d2h", "both"):
    for it in range(3):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        s2.wait_stream(torch.cuda.current_stream())
        if name in ("h2d", "both"):
            d.copy_(h, non_blocking=True)
        if name == "d2h":
            h.copy_(d, non_blocking=True)
        if name == "both":
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"{name}: {n / ms / 1e6:.1f} GB/s per direction ({ms:.2f} ms for {n >> 20} MiB)")
