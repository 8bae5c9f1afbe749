"""HBM write / copy bandwidth probe (the ceiling of output-bound layers)."""
import torch

n = 1 << 28  # 1 GiB of fp32
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
for name, fn, nbytes in (("zero_ (write only)", lambda: a.zero_(), 4 * n),
                         ("fill_ (write only)", lambda: a.fill_(1.0), 4 * n),
                         ("copy_ (read + write)", lambda: b.copy_(a), 8 * n)):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"{name:24s} {nbytes / ms / 1e6:8.0f} GB/s")
