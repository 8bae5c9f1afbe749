"""PCIe copy rate from page-locked memory vs. the number of streams per
direction (does one copy stream saturate the link, or the copy engine?).
Duplex: H2D and D2H at once, k streams each, the bytes split in equal chunks
over the streams.
    python tools/pcie_streams.py [MiB per direction]"""
import sys

import torch

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = (mib << 20) // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(mode, k, chunk_mib):
    cs = (chunk_mib << 20) // 4
    chunks = [(i, min(i + cs, n)) for i in range(0, n, cs)]
    main = torch.cuda.current_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(main)
    for s in streams:
        s.wait_stream(main)
    for j, (lo, hi) in enumerate(chunks):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(streams[j % k]):
                d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(streams[k + j % k] if mode == "both" else streams[j % k]):
                h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
    for s in streams:
        main.wait_stream(s)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for mode in ("h2d", "d2h", "both"):
    for k in (1, 2, 4):
        for chunk in (16, 64):
            best = min(run(mode, k, chunk) for _ in range(4))
            print(f"{mode:4s} streams/dir={k} chunk={chunk:3d} MiB: {mib / 1024 / best * 1e3:6.1f} GiB/s "
                  f"per direction ({best:.2f} ms)")
