"""Per-layer device time of the convolution kernel alone (filter prepared
once outside the timing, the run phase replayed from a CUDA graph, L2
flushed before every replay), for the VGG-16 and ResNet-50 layer tables.

    python tools/layer_times.py [vgg16|resnet50|all] [tf32|bf16] [batch] [--only NAME] [--io bf16]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1904_05347_b200 as tk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("which", nargs="?", default="all")
ap.add_argument("prec", nargs="?", default="tf32")
ap.add_argument("batch", nargs="?", type=int, default=32)
ap.add_argument("--only", default="")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--mode", default="auto", help="tensor-core operand path (tk.TC_MODES)")
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--algo", default="im2col", help="conv algorithm (parse_conv_params grammar)")
ap.add_argument("--io", default="fp32", help="activation format: fp32 | bf16 | in_bf16 | out_bf16 "
                                            "(bf16 needs the bf16 precision)")
ap.add_argument("--flush", default="read", choices=["read", "write"],
                help="evict L2 by reading (clean lines) or writing (dirty lines whose "
                     "write-back then lands on the timed kernel) a 256 MiB buffer")
a = ap.parse_args()

rows = []
if a.which in ("vgg16", "all"):
    rows += [(n, 3, 1, h, c, k) for n, h, c, k, _ in bench.VGG16]
if a.which in ("resnet50", "all"):
    rows += [(n, r, s, h, c, k) for n, r, s, h, c, k, _ in bench.RESNET50]
peaks, _ = bench.load_peaks()
peak = peaks["bf16_tflops"] / (2.0 if a.prec == "tf32" else 1.0)
flush = torch.ones(64 << 20, device="cuda")
flush_sink = torch.empty((), device="cuda")
p = tk.parse_conv_params(a.algo)
st = torch.cuda.Stream()
print(f"{'layer':18s} {'us':>8s} {'TF/s':>8s} {'%peak':>6s}  ({a.prec}, batch {a.batch}, peak {peak:.0f})")
for name, r, s, h, c, k in rows:
    if a.only and a.only not in name:
        continue
    shp = tk.ConvShape(a.batch, h, h, c, k, r, r, s, True)
    x = torch.rand(shp.in_shape, device="cuda") * 2 - 1
    f = torch.rand(shp.filt_shape, device="cuda") * 2 - 1
    y = torch.empty(shp.out_shape, device="cuda")
    if a.io in ("bf16", "in_bf16"):
        x = x.to(torch.bfloat16)
    if a.io in ("bf16", "out_bf16"):
        y = y.to(torch.bfloat16)
    opts = tk.exec_options(a.prec, mode=a.mode, split=a.split, io=a.io)
    try:
        ws = torch.empty(max(tk.conv2d_workspace_size(shp, p, options=opts), 4) // 4 + 1,
                         device="cuda")
    except tk.CapabilityError:
        print(f"{name:18s} {'n/a':>8s}")
        continue
    tk.conv2d_prepare_dev(f, shp, p, ws, stream=st, options=opts)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        tk.conv2d_run_dev(x, f, y, shp, p, ws, stream=st, options=opts)
    ts = []
    for i in range(a.reps + 2):
        if a.flush == "write":
            flush.zero_()
        else:
            flush_sink.copy_(flush.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(st):  # replay() launches on the current stream
            e0.record(st)
            g.replay()
            e1.record(st)
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    us = float(np.median(ts)) * 1e3
    tf = shp.flops() / (us * 1e-6) / 1e12
    print(f"{name:18s} {us:8.1f} {tf:8.1f} {100 * tf / peak:5.1f}%", flush=True)
