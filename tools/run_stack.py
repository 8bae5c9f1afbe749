"""Run the ResNet-50 (or VGG-16) conv stack once, layer by layer, for ncu
launch lists.  python tools/run_stack.py resnet50|vgg16 [tf32|bf16] [batch]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1904_05347_b200 as tk  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
prec = sys.argv[2] if len(sys.argv) > 2 else "tf32"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 32
rows = ([(n, r, s, h, c, k, m) for n, r, s, h, c, k, m in bench.RESNET50] if which == "resnet50"
        else [(n, 3, 1, h, c, k, m) for n, h, c, k, m in bench.VGG16])
p = tk.parse_conv_params("im2col")
for it in range(2):
    for name, r, s, h, c, k, m in rows:
        shp = tk.ConvShape(N, h, h, c, k, r, r, s, True)
        x = torch.rand(shp.in_shape, device="cuda")
        f = torch.rand(shp.filt_shape, device="cuda")
        y = torch.empty(shp.out_shape, device="cuda")
        ws = torch.empty(tk.conv2d_workspace_size(shp, p, prec) // 4 + 1, device="cuda")
        torch.cuda.synchronize()
        tk.conv2d_dev(x, f, y, shp, p, precision=prec, workspace=ws)
        torch.cuda.synchronize()
print("ok")
