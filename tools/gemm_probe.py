"""Tensor-core GEMM probe: C = A^T B with both operands K-major in place (no
packing), graph-replayed, for several tile widths.
    python tools/gemm_probe.py M,N,K[;M,N,K...] [tf32|bf16]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05347_b200 as tk  # noqa: E402

shapes = [tuple(int(v) for v in t.split(",")) for t in
          (sys.argv[1] if len(sys.argv) > 1 else "2048,2048,2048;8192,8192,8192").split(";")]
prec = sys.argv[2] if len(sys.argv) > 2 else "tf32"
st = torch.cuda.Stream()
for m, n, k in shapes:
    a = torch.rand(m * k, device="cuda") - 0.5
    b = torch.rand(k * n, device="cuda") - 0.5
    c = torch.empty(m * n, device="cuda")
    shape = tk.GemmShape(m, n, k, 1.0, 0.0, os.environ.get("TA", "t"), "n")
    for tn in (0, 64, 128, 256):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(5):
                tk.gemm_dev(a, b, None, c, shape, None, precision=prec, stream=st, tile_n=tn)
        with torch.cuda.stream(st):
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 5
        print(f"{m}x{n}x{k} {prec} tile_n={tn}: {us:8.1f} us {2 * m * n * k / us / 1e6:8.1f} TF/s",
              flush=True)
