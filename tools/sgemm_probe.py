"""SGEMM call-path probe (BASELINE configs[0], 1024^3 column-major nn with
the row-major operands swapped): per precision, (a) the event time of one
API call as bench.py takes it, (b) device time from a CUDA graph of 20 calls
(no host work), (c) host time per call (1000 back-to-back calls).
    python tools/sgemm_probe.py [n] [tile_n/cluster[/split],...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05347_b200 as tk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tiles = [tuple(int(x) for x in v.split("/")) + (0,) * (3 - len(v.split("/")))
         for v in sys.argv[2].split(",")] \
    if len(sys.argv) > 2 else [(0, 0, 0)]  # tile_n/cluster[/split] triples
a = torch.rand(n * n, device="cuda") * 2 - 1
b = torch.rand(n * n, device="cuda") * 2 - 1
c = torch.empty(n * n, device="cuda")
shape = tk.GemmShape(n, n, n)
st = torch.cuda.Stream()
fl = 2 * n ** 3
for prec in ("fp32", "tf32", "bf16", "3xtf32"):
    for tn, cl, sp in (tiles if prec in ("tf32", "bf16") else [(0, 0, 0)]):
        opts = tk.exec_options(prec, tile_n=tn, cluster=cl, split=sp)

        def call(s=st):
            tk.gemm_dev(b, a, None, c, shape, None, stream=s, options=opts)
        with torch.cuda.stream(st):
            for _ in range(3):
                call()
            st.synchronize()
            ev = []
            for _ in range(20):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                call()
                e1.record(st)
                e1.synchronize()
                ev.append(e0.elapsed_time(e1) * 1e3)
            reps = 20
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(reps):
                    call()
            g.replay()
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            e1.synchronize()
            dev_us = e0.elapsed_time(e1) * 1e3 / reps
            t0 = time.perf_counter()
            for _ in range(200):
                call()
            host_us = (time.perf_counter() - t0) / 200 * 1e6
            st.synchronize()
        print(f"{n}^3 {prec:6s} tile_n={tn:3d} cg={cl} split={sp}: api(event) {np.median(ev):7.1f} us  "
              f"device(graph) {dev_us:7.1f} us = {fl / dev_us / 1e6:7.1f} TF/s  "
              f"host/call {host_us:6.1f} us", flush=True)
