"""Launch-floor probe: graph-replayed run phase of tiny and small 1x1 layers."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05347_b200 as tk  # noqa: E402

p = tk.parse_conv_params("im2col")
st = torch.cuda.Stream()
CASES = [(1, 7, 64, 64, 1), (1, 14, 256, 256, 1), (32, 7, 2048, 512, 1),
         (32, 7, 512, 2048, 1), (32, 14, 1024, 256, 1), (1, 7, 64, 64, 3)]
if len(sys.argv) > 1:
    CASES = [tuple(int(v) for v in sys.argv[1].split(","))]
for (n, h, c, k, r) in CASES:
    for prec in ("tf32",):
        shp = tk.ConvShape(n, h, h, c, k, r, r, 1, True)
        x = torch.rand(shp.in_shape, device="cuda")
        f = torch.rand(shp.filt_shape, device="cuda")
        y = torch.empty(shp.out_shape, device="cuda")
        ws = torch.empty(max(tk.conv2d_workspace_size(shp, p, prec), 4) // 4 + 1, device="cuda")
        tk.conv2d_prepare_dev(f, shp, p, ws, precision=prec, stream=st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(10):
                tk.conv2d_run_dev(x, f, y, shp, p, ws, precision=prec, stream=st)
        with torch.cuda.stream(st):
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
        e1.synchronize()
        print(f"N={n} {h}x{h}x{c}->{k} r={r} {prec}: {e0.elapsed_time(e1) * 100:.1f} us per call "
              f"(10 back-to-back in a graph)")
