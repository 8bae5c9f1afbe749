"""Where does the VGG16 step time go beyond the sum of its kernels?
Times (CUDA events, L2 written between replays like bench.py) the step graph
in variants: full (prepares on a side stream + runs), runs only (filters
prepared beforehand), and runs with an L2 eviction between layers.
    python tools/step_probe.py [tf32|bf16]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1904_05347_b200 as tk  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "tf32"
N = 32
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(1234)
algo = tk.parse_conv_params("im2col")
layers = []
for name, h, c, k, mult in bench.VGG16:
    for _ in range(mult):
        shape = tk.ConvShape(N, h, h, c, k, 3, 3, 1, True)
        x = torch.rand((N, h, h, c), device=dev, generator=gen) * 2 - 1
        f = torch.rand((3, 3, c, k), device=dev, generator=gen) * 2 - 1
        y = torch.empty((N, h, h, k), device=dev)
        ws = torch.empty(max(tk.conv2d_workspace_size(shape, algo, prec), 4) // 4 + 1, device=dev)
        tk.conv2d_prepare_dev(f, shape, algo, ws, precision=prec)
        layers.append((name, shape, x, f, y, ws))
flush = torch.empty(64 << 20, device=dev)
sink = torch.empty((), device=dev)
torch.cuda.synchronize()


def graph_of(body):
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        body(st)
    return g


def timeit(g, n=10, pre=lambda: flush.zero_(), spread=False):
    ts = []
    for _ in range(n + 2):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    t = np.array(ts[2:])
    if spread:
        return f"min {t.min():.3f} med {np.median(t):.3f} mean {t.mean():.3f} max {t.max():.3f}"
    return float(np.median(t))


def runs(st):
    for name, shape, x, f, y, ws in layers:
        tk.conv2d_run_dev(x, f, y, shape, algo, ws, precision=prec, stream=st)


def full(st):
    side = torch.cuda.Stream()
    side.wait_stream(st)
    evs = []
    with torch.cuda.stream(side):
        for name, shape, x, f, y, ws in layers:
            tk.conv2d_prepare_dev(f, shape, algo, ws, precision=prec, stream=side)
            e = torch.cuda.Event()
            e.record(side)
            evs.append(e)
    for (name, shape, x, f, y, ws), e in zip(layers, evs):
        st.wait_event(e)
        tk.conv2d_run_dev(x, f, y, shape, algo, ws, precision=prec, stream=st)
    st.wait_stream(side)


def prep_first(st):
    for name, shape, x, f, y, ws in layers:
        tk.conv2d_prepare_dev(f, shape, algo, ws, precision=prec, stream=st)
    runs(st)


for nm, body in (("full", full), ("prepares first", prep_first), ("runs only", runs)):
    g = graph_of(body)
    print(f"{nm:16s} x50: {timeit(g, n=50, spread=True)}", flush=True)
gf = graph_of(full)
for nm, pre in (("write flush", lambda: flush.zero_()),
                ("read evict", lambda: torch.sum(flush, dim=0, out=sink)),
                ("no eviction", lambda: None)):
    print(f"full, {nm:12s} x100: {timeit(gf, n=100, pre=pre, spread=True)}", flush=True)
print(f"full step            {timeit(graph_of(full)):8.3f} ms")
print(f"runs only            {timeit(graph_of(runs)):8.3f} ms")
print(f"runs only, read-evict{timeit(graph_of(runs), pre=lambda: torch.sum(flush, dim=0, out=sink)):8.3f} ms")
tot = 0.0
for L in layers:
    name, shape, x, f, y, ws = L
    g = graph_of(lambda st, L=L: tk.conv2d_run_dev(L[2], L[3], L[4], L[1], algo, L[5],
                                                    precision=prec, stream=st))
    t = timeit(g, n=5)
    tot += t
    print(f"  {name:14s} single replay {t * 1e3:8.1f} us")
print(f"sum of single replays {tot:8.3f} ms")
