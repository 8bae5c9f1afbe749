"""Where does a layer's event-timed time go?  Times one conv layer run phase
(direct launch vs graph replay, with and without an L2 eviction before it)
and a trivial kernel the same ways.
    python tools/overhead_probe.py N,H,C,K,R [tf32|bf16]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05347_b200 as tk  # noqa: E402

N, H, C, K, R = (int(v) for v in sys.argv[1].split(","))
prec = sys.argv[2] if len(sys.argv) > 2 else "tf32"
shp = tk.ConvShape(N, H, H, C, K, R, R, 1, True)
p = tk.parse_conv_params("im2col")
x = torch.rand(shp.in_shape, device="cuda")
f = torch.rand(shp.filt_shape, device="cuda")
y = torch.empty(shp.out_shape, device="cuda")
ws = torch.empty(max(tk.conv2d_workspace_size(shp, p, prec), 4) // 4 + 1, device="cuda")
st = torch.cuda.Stream()
tk.conv2d_prepare_dev(f, shp, p, ws, precision=prec, stream=st)
st.synchronize()
flush = torch.ones(64 << 20, device="cuda")
sink = torch.empty((), device="cuda")
small = torch.zeros(1, device="cuda")


def run():
    tk.conv2d_run_dev(x, f, y, shp, p, ws, precision=prec, stream=st)


def triv():
    with torch.cuda.stream(st):
        small.add_(1)


def timeit(fn, do_flush, graph):
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        fn2 = g.replay
    else:
        fn2 = fn
    ts = []
    for i in range(12):
        if do_flush:
            sink.copy_(flush.sum())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            fn2()
            e1.record(st)
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for name, fn in (("conv", run), ("trivial", triv)):
    for graph in (False, True):
        for fl in (False, True):
            print(f"{name:8s} graph={graph!s:5s} flush={fl!s:5s} {timeit(fn, fl, graph):8.1f} us",
                  flush=True)
# back-to-back replays: 10 launches between one pair of events
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st)
    for _ in range(10):
        g.replay()
    e1.record(st)
e1.synchronize()
print(f"conv 10 back-to-back replays: {e0.elapsed_time(e1) * 100:.1f} us each")
