"""Max scaled error of the TF32 conv path vs the oracle on VGG/ResNet shapes
(one image checked per shape)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1904_05347_b200 as tk  # noqa: E402
import pyoracle as O  # noqa: E402

shapes = [(224, 64, 64, 3, 1), (112, 128, 128, 3, 1), (56, 256, 256, 3, 1), (28, 512, 512, 3, 1),
          (14, 512, 512, 3, 1), (56, 64, 256, 1, 1), (14, 1024, 256, 1, 1), (7, 2048, 512, 1, 1)]
for seed in (1, 2):
    for h, c, k, r, st in shapes:
        s = tk.ConvShape(2, h, h, c, k, r, r, st, True)
        conv = O.Conv(2, h, h, c, k, r, r, st, True)
        x = O.fill_random(int(np.prod(conv.in_shape)), seed).reshape(conv.in_shape)
        f = O.fill_random(int(np.prod(conv.filt_shape)), seed + 7).reshape(conv.filt_shape)
        want = O.conv2d_naive(conv, x, f)
        dy = torch.empty(conv.out_shape, device="cuda")
        tk.conv2d_dev(torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda(), dy, s,
                      tk.parse_conv_params("im2col"), precision="tf32")
        torch.cuda.synchronize()
        print(f"seed{seed} {h}x{c}->{k} r{r}: scaled {O.max_scaled_error(dy.cpu().numpy(), want):.2e}",
              flush=True)
