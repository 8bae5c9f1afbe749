"""Generate golden fixtures from the UNMODIFIED reference (run in the build
container, where /root/reference exists).

    python tests/golden/make_golden.py

Builds oracle/_ref/libtkref.so (oracle/ref_shim.cpp compiled straight from
/root/reference/proj/include) and records the reference's own outputs:

* rng.npz      -- tuner.hpp:293-297 fill_random for several seeds
* gemm.npz     -- gemm_naive on the test_gemm.cpp shape grid (tails, every
                  op combination, alpha/beta corners) with seeded inputs
* conv.npz     -- conv2d_naive / im2col on a randomized shape grid in the
                  spirit of acceptance.cpp criterion 3 (stride 1/2, Same and
                  Valid, 1x1/3x3/7x7 windows) plus conv2d_winograd F(2x2)
                  and F(4x4) outputs and WinogradStats
Inputs are regenerated from the stored seeds with the (pinned) fill_random,
so only outputs are stored.  The GPU box never runs this script.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as O  # noqa: E402


def gemm_cases():
    cases = []
    for m in (1, 2, 3, 16, 32, 33, 64, 67):          # test_gemm.cpp:252-272
        for n in (1, 32, 45):
            for k in (1, 17, 64):
                cases.append(dict(m=m, n=n, k=k, alpha=1.5, beta=-0.5, ta=0, tb=0,
                                  seed=100 + m * 7 + n * 3 + k))
    for ta in (0, 1):                                    # test_gemm.cpp:274-291
        for tb in (0, 1):
            for alpha, beta in ((1.0, 1.0), (0.0, 1.0), (1.0, 0.0), (0.5, -1.0)):
                cases.append(dict(m=33, n=29, k=21, alpha=alpha, beta=beta, ta=ta, tb=tb,
                                  seed=17 + ta * 2 + tb))
    cases.append(dict(m=96, n=80, k=70, alpha=1.0, beta=1.0, ta=0, tb=0, seed=5))  # :305-322
    cases.append(dict(m=130, n=70, k=50, alpha=1.0, beta=0.5, ta=0, tb=0, seed=8))  # :349-364
    cases.append(dict(m=257, n=129, k=300, alpha=0.5, beta=-1.0, ta=1, tb=0, seed=20240811))
    return cases


def gemm_inputs(c):
    m, n, k = c["m"], c["n"], c["k"]
    a = O.fill_random(m * k, c["seed"])
    b = O.fill_random(k * n, c["seed"] + 1)
    cc = O.fill_random(m * n, c["seed"] + 2)
    return a, b, cc


def conv_cases():
    rng = np.random.default_rng(42)
    cases = []
    while len(cases) < 60:
        s = dict(batch=int(rng.integers(1, 3)), in_rows=int(rng.integers(4, 13)),
                 in_cols=int(rng.integers(4, 13)), channels=int(rng.choice([1, 3, 8, 16])),
                 features=int(rng.choice([1, 3, 8, 20])), window=int(rng.choice([1, 3, 3, 7])),
                 stride=int(rng.integers(1, 3)), same=bool(rng.integers(0, 2)))
        conv = to_conv(s)
        if conv.out_rows == 0 or conv.out_cols == 0:
            continue
        s["seed"] = 1000 + len(cases)
        cases.append(s)
    # Fixed shapes: the reference test_conv.cpp cases and a VGG-like layer.
    for s in (dict(batch=1, in_rows=9, in_cols=7, channels=8, features=4, window=3, stride=1, same=True),
              dict(batch=2, in_rows=12, in_cols=10, channels=6, features=8, window=3, stride=2, same=False),
              dict(batch=2, in_rows=7, in_cols=7, channels=4, features=3, window=3, stride=1, same=True),
              dict(batch=1, in_rows=28, in_cols=28, channels=32, features=64, window=3, stride=1, same=True),
              dict(batch=2, in_rows=23, in_cols=23, channels=3, features=16, window=7, stride=2, same=True),
              dict(batch=1, in_rows=14, in_cols=14, channels=64, features=32, window=1, stride=2, same=True)):
        s["seed"] = 1000 + len(cases)
        cases.append(s)
    return cases


def to_conv(s) -> O.Conv:
    return O.Conv(s["batch"], s["in_rows"], s["in_cols"], s["channels"], s["features"],
                  s["window"], s["window"], s["stride"], s["same"])


def conv_inputs(s):
    c = to_conv(s)
    i = O.fill_random(int(np.prod(c.in_shape)), s["seed"]).reshape(c.in_shape)
    f = O.fill_random(int(np.prod(c.filt_shape)), s["seed"] + 1).reshape(c.filt_shape)
    return c, i, f


def main() -> None:
    O.build()
    if not O.have_ref():
        sys.exit("reference not built; /root/reference is required")

    seeds = [0, 1, 42, 20240811, 0x9E3779B97F4A7C15]
    np.savez_compressed(os.path.join(HERE, "rng.npz"), seeds=np.array(seeds, np.uint64),
                        values=np.stack([O.ref_fill_random(256, s) for s in seeds]))

    gc = gemm_cases()
    outs = {}
    for i, c in enumerate(gc):
        a, b, cc = gemm_inputs(c)
        outs[f"out{i}"] = O.ref_gemm_naive(c["m"], c["n"], c["k"], c["alpha"], c["beta"],
                                           c["ta"], c["tb"], a, b, cc)
    np.savez_compressed(os.path.join(HERE, "gemm.npz"), meta=json.dumps(gc), **outs)

    cc_ = conv_cases()
    outs = {}
    for i, s in enumerate(cc_):
        conv, x, f = conv_inputs(s)
        outs[f"naive{i}"] = O.ref_conv2d(conv, "naive", x, f)
        outs[f"im2col{i}"] = O.ref_im2col(conv, x)
        if conv.window_rows == 3 and conv.stride == 1:
            for m in (2, 4):
                w, mults, tiles = O.ref_conv2d_winograd(conv, m, x, f)
                outs[f"wino{m}_{i}"] = w
                s[f"wino{m}_stats"] = [mults, tiles]
    np.savez_compressed(os.path.join(HERE, "conv.npz"), meta=json.dumps(cc_), **outs)
    for fn in ("rng.npz", "gemm.npz", "conv.npz"):
        print(fn, os.path.getsize(os.path.join(HERE, fn)), "bytes")


if __name__ == "__main__":
    main()
