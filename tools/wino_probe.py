"""One Winograd conv2d_dev call per (layer, m, precision), for an ncu launch
list of its transform / batched-GEMM kernels.
    python tools/wino_probe.py [layer] [warm]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05347_b200 as tk  # noqa: E402
from bench import VGG16  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vgg_conv4_2"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
h, c, k = [(hh, cc, kk) for n, hh, cc, kk, _ in VGG16 if n == name][0]
shp = tk.ConvShape(32, h, h, c, k, 3, 3, 1, True)
x = torch.rand(shp.in_shape, device="cuda") * 2 - 1
f = torch.rand(shp.filt_shape, device="cuda") * 2 - 1
y = torch.empty(shp.out_shape, device="cuda")
for algo, prec in (("winograd_t2x2", "tf32"), ("winograd_t4x4", "tf32"), ("winograd_t4x4", "3xtf32"),
                   ("im2col", "tf32")):
    p = tk.parse_conv_params(algo)
    ws = torch.empty(tk.conv2d_workspace_size(shp, p, prec) // 4 + 1, device="cuda")
    for _ in range(warm + 1):
        tk.conv2d_dev(x, f, y, shp, p, precision=prec, workspace=ws)
    torch.cuda.synchronize()
    print(algo, prec, "ok", flush=True)
