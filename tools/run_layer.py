"""Run one conv layer through the C ABI (device buffers) for profiling.

    python tools/run_layer.py --h 28 --c 512 --k 512 --batch 32 --algo im2col --prec tf32 --iters 3
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05347_b200 as tk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--h", type=int, default=28)
ap.add_argument("--c", type=int, default=512)
ap.add_argument("--k", type=int, default=512)
ap.add_argument("--r", type=int, default=3)
ap.add_argument("--stride", type=int, default=1)
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--algo", default="im2col")
ap.add_argument("--prec", default="tf32")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--tile-n", type=int, default=0)
a = ap.parse_args()
s = tk.ConvShape(a.batch, a.h, a.h, a.c, a.k, a.r, a.r, a.stride, True)
p = tk.parse_conv_params(a.algo)
x = torch.rand(s.in_shape, device="cuda") * 2 - 1
f = torch.rand(s.filt_shape, device="cuda") * 2 - 1
y = torch.empty(s.out_shape, device="cuda")
ws = torch.empty(tk.conv2d_workspace_size(s, p, a.prec) // 4 + 1, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(a.iters):
    ev[0].record()
    tk.conv2d_dev(x, f, y, s, p, precision=a.prec, workspace=ws, tile_n=a.tile_n)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    print(f"iter {i}: {ms:.4f} ms  {s.flops() / ms / 1e9:.1f} TFLOP/s")
