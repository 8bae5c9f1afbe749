"""One small launch of every kernel mode, for compute-sanitizer.

    compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck --error-exitcode 1 python tools/sanitize_cases.py

Covers the hand-written mbarrier / TMEM / TMA pipelines (halo, pixN incl.
multi-image and flat-row tiles and split-K, pixM, gather, pointwise,
im2col-mode TMA, stream-K tail), the exact SIMT family, Winograd and the
tensor-core GEMMs (K-major and MN-major A), in TF32 and BF16.  Each result
is also compared against the oracle so a sanitizer run doubles as a parity
smoke test.  `--only NAME` runs one case.  `--bench` adds every bench.py
layer shape at batch 32 (TF32, BF16, BF16 with bf16 activations) through the
bench's plans, checked for finite outputs -- run against the checked build
(`TK_LIB_PATH=paper_1904_05347_b200/libtilekit_b200_checked.so`, device-side
invariants on) by tests/test_gpu_checked.py, since compute-sanitizer itself
is closed on this GPU pool.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

# (name, N, H, C, K, R, stride, algo, mode, precisions)
CONV_CASES = [
    ("halo", 2, 28, 64, 64, 3, 1, "im2col", "halo", ("tf32", "bf16")),
    ("pixn", 2, 14, 256, 256, 3, 1, "im2col", "pixn", ("tf32", "bf16")),
    ("pixn_multi_image_split", 8, 7, 256, 512, 3, 1, "im2col", "auto", ("tf32",)),
    ("pixm", 2, 20, 64, 64, 3, 1, "im2col", "pixm", ("tf32",)),
    ("gather_c3", 2, 30, 3, 64, 3, 1, "im2col", "auto", ("tf32",)),
    ("gather_stem", 1, 40, 3, 64, 7, 2, "im2col", "auto", ("tf32",)),
    ("pointwise", 4, 14, 256, 256, 1, 1, "im2col", "pointwise", ("tf32", "bf16")),
    ("im2col_tma", 2, 28, 128, 256, 3, 1, "im2col", "im2col", ("tf32", "bf16")),
    ("im2col_s2", 2, 28, 256, 512, 1, 2, "im2col", "auto", ("tf32",)),
    ("exact", 1, 14, 32, 48, 3, 1, "tiled_t4x4_v4x4", "auto", ("fp32",)),
    ("winograd_f2", 1, 16, 64, 64, 3, 1, "winograd_t2x2", "auto", ("tf32", "fp32")),
    ("winograd_f4", 1, 16, 64, 64, 3, 1, "winograd_t4x4", "auto", ("tf32",)),
]
GEMM_CASES = [  # (name, m, n, k, op_a, op_b, precision)
    ("gemm_kmajor", 256, 192, 100, "t", "n", "tf32"),
    ("gemm_mn_major_a", 256, 256, 70, "n", "n", "tf32"),
    ("gemm_bf16", 300, 200, 128, "n", "t", "bf16"),
    ("gemm_3xtf32", 128, 128, 64, "n", "n", "3xtf32"),
    ("gemm_exact", 67, 45, 17, "n", "n", "fp32"),
    ("gemm_tail", 1024, 1024, 1024, "n", "n", "tf32"),
]
TOL = {"tf32": 1e-3, "bf16": 5e-3, "3xtf32": 5e-5, "fp32": 0.0}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--bench", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_1904_05347_b200 as tk
    import pyoracle as O

    bad = 0
    for name, n, h, c, k, r, st, algo, mode, precs in CONV_CASES:
        if args.only and args.only != name:
            continue
        s = tk.ConvShape(n, h, h, c, k, r, r, st, True)
        conv = O.Conv(n, h, h, c, k, r, r, st, True)
        x = O.fill_random(int(np.prod(conv.in_shape)), 3).reshape(conv.in_shape)
        f = O.fill_random(int(np.prod(conv.filt_shape)), 4).reshape(conv.filt_shape)
        want = O.conv2d_naive(conv, x, f)
        for p in precs:
            params = tk.parse_conv_params(algo)
            opts = tk.exec_options(p, mode=mode)
            ws = torch.empty(max(tk.conv2d_workspace_size(s, params, options=opts), 4) // 4 + 1,
                             device="cuda")
            y = torch.full(s.out_shape, float("nan"), device="cuda")
            tk.conv2d_dev(torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda(), y, s, params,
                          workspace=ws, options=opts)
            torch.cuda.synchronize()
            got = y.cpu().numpy()
            err = O.max_scaled_error(got, want)
            # (exact FP32 Winograd is bit-identical to the reference's Winograd,
            # tested bit for bit in the GPU suite -- not to the direct sum checked here)
            tol = 1e-2 if algo == "winograd_t4x4" else (1e-5 if algo.startswith("winograd") and
                                                         p == "fp32" else TOL[p])
            ok = err <= tol and not np.isnan(got).any()
            bad += not ok
            print(f"{name:24s} {p:6s} err={err:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    for name, m, nn, kk, oa, ob, p in GEMM_CASES:
        if args.only and args.only != name:
            continue
        a = O.fill_random(m * kk, 1)
        b = O.fill_random(kk * nn, 2)
        want = O.gemm_naive(m, nn, kk, 1.0, 0.0, int(oa == "t"), int(ob == "t"), a, b,
                            np.zeros(m * nn, np.float32))
        out = torch.full((m * nn,), float("nan"), device="cuda")
        tk.gemm_dev(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), None, out,
                    tk.GemmShape(m, nn, kk, 1.0, 0.0, oa, ob), precision=p)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        err = O.max_scaled_error(got, want)
        ok = err <= TOL[p] and not np.isnan(got).any()
        bad += not ok
        print(f"{name:24s} {p:6s} err={err:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    if args.bench:
        from bench import RESNET50, VGG16
        layers = [(n, 3, 1, h, c, k) for n, h, c, k, _ in VGG16] + \
                 [(n, r, st, h, c, k) for n, r, st, h, c, k, _ in RESNET50]
        im = tk.parse_conv_params("im2col")
        for name, r, st, h, c, k in layers:
            s = tk.ConvShape(32, h, h, c, k, r, r, st, True)
            x = torch.rand(s.in_shape, device="cuda") * 2 - 1
            f = torch.rand(s.filt_shape, device="cuda") * 2 - 1
            for p, io in (("tf32", "fp32"), ("bf16", "fp32"), ("bf16", "bf16")):
                opts = tk.exec_options(p, io=io)
                xi = x.to(torch.bfloat16) if io == "bf16" else x
                y = torch.full(s.out_shape, float("nan"), device="cuda",
                               dtype=torch.bfloat16 if io == "bf16" else torch.float32)
                tk.conv2d_dev(xi, f, y, s, im, options=opts)
                torch.cuda.synchronize()
                ok = bool(torch.isfinite(y.float()).all())
                bad += not ok
                print(f"bench {name:18s} {p}/{io:5s} {'ok' if ok else 'FAIL (non-finite)'}", flush=True)
    print("FAILED" if bad else "all ok", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
