"""Exact FP32 path probe: device time (graph of reps calls) of conv layers
through several conv2d algorithms / tiled params, and SGEMM with GemmConfigs.
    python tools/exact_probe.py [layer,...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05347_b200 as tk  # noqa: E402
from bench import VGG16, RESNET50  # noqa: E402

st = torch.cuda.Stream()


def dev_ms(fn, reps=3):
    with torch.cuda.stream(st):
        fn()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
    return e0.elapsed_time(e1) / reps


want = sys.argv[1].split(",") if len(sys.argv) > 1 else ["vgg_conv3_2", "vgg_conv1_1", "conv1",
                                                          "res2a_branch2a", "res4a_branch2b"]
rows = {n: (3, 1, h, c, k) for n, h, c, k, _ in VGG16}
rows.update({n: (r, s, h, c, k) for n, r, s, h, c, k, _ in RESNET50})
for name in want:
    r, s, h, c, k = rows[name]
    shp = tk.ConvShape(32, h, h, c, k, r, r, s, True)
    x = torch.rand(shp.in_shape, device="cuda") * 2 - 1
    f = torch.rand(shp.filt_shape, device="cuda") * 2 - 1
    y = torch.empty(shp.out_shape, device="cuda")
    for algo in ("naive", "tiled_t4x5_v4x2", "tiled_t4x4_v4x4", "tiled_t2x4_v4x8", "tiled_t1x8_v4x8",
                 "tiled_t4x2_v4x8", "tiled_t2x2_v4x8", "tiled_t8x1_v4x8", "tiled_t8x4_v4x4"):
        pa = tk.parse_conv_params(algo)
        ms = dev_ms(lambda: tk.conv2d_dev(x, f, y, shp, pa, precision="fp32", stream=st))
        print(f"{name:16s} {algo:18s} {ms:8.3f} ms {shp.flops() / ms / 1e9:7.2f} TF/s "
              f"[{tk.conv2d_plan_info(shp, pa, 'fp32')['tile_m']}x"
              f"{tk.conv2d_plan_info(shp, pa, 'fp32')['tile_n']}]", flush=True)
n = 1024
a = torch.rand(n * n, device="cuda") * 2 - 1
b = torch.rand(n * n, device="cuda") * 2 - 1
cc = torch.empty(n * n, device="cuda")
for cfg in (None, "8x8_16x16_loc_db", "8x4_8x16_loc", "4x4_16x16_loc_db", "8x8_8x16_loc_db",
            "4x8_16x8_loc_db", "8x4_16x8_loc_db", "3x5_8x8_loc", "6x6_16x8_loc_db"):
    gc = tk.parse_gemm_config(cfg) if cfg else None
    ms = dev_ms(lambda: tk.gemm_dev(b, a, None, cc, tk.GemmShape(n, n, n), gc, precision="fp32",
                                    stream=st), reps=10)
    print(f"sgemm1024 {str(cfg):18s} {ms * 1e3:8.1f} us {2 * n ** 3 / ms / 1e9:7.2f} TF/s", flush=True)
