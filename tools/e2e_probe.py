"""A/B of the host-buffer pipeline (tk_conv2d_ex, pinned host memory) on
the bench's VGG16 step: each knob value in its own process.
    python tools/e2e_probe.py TK_PIPE_CHUNKS 8,16,32 [precision]"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "--worker":
    import ctypes
    sys.path.insert(0, ROOT)
    import torch
    import paper_1904_05347_b200 as tk
    from bench import VGG16
    prec = sys.argv[2]
    im = tk.parse_conv_params("im2col")
    seq, flops = [], 0.0
    for name, h, c, k, mult in VGG16:
        s = tk.ConvShape(32, h, h, c, k, 3, 3, 1, True)
        hb = dict(s=s, x=(torch.rand(s.in_shape) * 2 - 1).pin_memory().numpy(),
                  f=(torch.rand(s.filt_shape) * 2 - 1).pin_memory().numpy(),
                  y=torch.empty(s.out_shape).pin_memory().numpy())
        seq += [hb] * mult
        flops += s.flops() * mult
    lib, opts = tk.lib(), tk.exec_options(prec)

    def step():
        for hb in seq:
            tk._check(lib.tk_conv2d_ex(ctypes.byref(hb["s"].c()), ctypes.byref(im.c()), ctypes.byref(opts),
                                       hb["x"].ctypes.data_as(ctypes.c_void_p),
                                       hb["f"].ctypes.data_as(ctypes.c_void_p),
                                       hb["y"].ctypes.data_as(ctypes.c_void_p)))
    step()
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(json.dumps({"ms_median": round(ts[len(ts) // 2] * 1e3, 2), "ms_min": round(ts[0] * 1e3, 2),
                      "gflops": round(flops / ts[len(ts) // 2] / 1e9, 1)}))
    sys.exit(0)

knob, values = sys.argv[1], sys.argv[2].split(",")
prec = sys.argv[3] if len(sys.argv) > 3 else "tf32"
for v in values:
    env = dict(os.environ, TK_EXPERIMENTS="1", **({knob: v} if v != "default" else {}))
    r = subprocess.run([sys.executable, __file__, "--worker", prec], env=env, capture_output=True,
                       text=True)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    print(f"{knob}={v}: {line[-1] if line else r.stderr[-400:]}", flush=True)
