"""GPU parity of the exact FP32 paths (bit-identical to the reference).

Every comparison here is on raw float bits: the SIMT kernels reproduce the
reference's ascending-k FMUL+FADD recurrence, so the
only acceptable max_rel_error is 0.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
STOCK = ["4x4_8x8_loc", "4x4_16x16_loc", "8x4_8x16_loc", "8x2_4x16_loc", "8x4_8x16_noloc",
         "8x4_4x8_noloc", "4x4_8x8_noloc"]


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def same(a, b):
    return np.array_equal(bits(a).ravel(), bits(b).ravel())


@pytest.fixture(scope="module")
def gpu_dev(tk):
    return tk.find_device("Intel Core i7-6700K GPU")


def test_gemm_golden_all_stock_configs(tk, oracle, gpu_dev):
    g = np.load(os.path.join(GOLDEN, "gemm.npz"))
    b200 = tk.b200_device()
    for i, c in enumerate(json.loads(str(g["meta"]))):
        m, n, k = c["m"], c["n"], c["k"]
        a = oracle.fill_random(m * k, c["seed"])
        b = oracle.fill_random(k * n, c["seed"] + 1)
        cc = oracle.fill_random(m * n, c["seed"] + 2)
        shape = tk.GemmShape(m, n, k, c["alpha"], c["beta"], "t" if c["ta"] else "n",
                             "t" if c["tb"] else "n")
        for name in STOCK + ["8x8_16x16_loc_db", "1x1_4x4_loc", "2x8_16x4_loc_db"]:
            dev = b200 if name.startswith(("8x8", "2x8")) else gpu_dev
            got = tk.gemm_tiled(a, b, cc, shape, tk.parse_gemm_config(name), dev)
            assert same(got, g[f"out{i}"]), (c, name)
        assert same(tk.gemm_naive(a, b, cc, shape), g[f"out{i}"]), c


def test_gemm_beta_zero_never_reads_c(tk, gpu_dev):
    shape = tk.GemmShape(1, 1, 1)
    for name in ["4x4_8x8_loc", "4x4_8x8_noloc", "8x4_8x16_loc_db"]:
        out = tk.gemm_tiled(np.array([3.0]), np.array([7.0]), np.array([np.nan]), shape,
                            tk.parse_gemm_config(name), gpu_dev)
        assert out[0] == 21.0


def test_gemm_1024_cube_bit_exact(tk, oracle):
    """Config 1 of BASELINE.json: SGEMM 1024^3, row-major C = A B realised as
    the column-major nn call with operands swapped."""
    n = 1024
    a = oracle.fill_random(n * n, 11)
    b = oracle.fill_random(n * n, 12)
    want = oracle.gemm_naive(n, n, n, 1.0, 0.0, 0, 0, b, a, None)   # (A B)^T col-major
    shape = tk.GemmShape(n, n, n)
    got = tk.gemm_tiled(b, a, None, shape, tk.parse_gemm_config("8x8_16x16_loc_db"),
                        tk.b200_device())
    assert same(got, want)
    assert oracle.max_rel_error(got, want) == 0.0


def test_gemm_batched_strided(tk, oracle):
    a = oracle.fill_random(16 * 37 * 19, 1)
    b = oracle.fill_random(16 * 19 * 23, 2)
    got, cnt = tk.gemm_batched_strided(a, b, 16, 37, 23, 19)
    want, wcnt = oracle.gemm_batched_strided(a, b, 16, 37, 23, 19)
    assert cnt == wcnt and same(got, want)


def conv_case(tk, oracle, s):
    shape = tk.ConvShape(s["batch"], s["in_rows"], s["in_cols"], s["channels"], s["features"],
                         s["window"], s["window"], s["stride"], s["same"])
    x = oracle.fill_random(int(np.prod(shape.in_shape)), s["seed"]).reshape(shape.in_shape)
    f = oracle.fill_random(int(np.prod(shape.filt_shape)), s["seed"] + 1).reshape(shape.filt_shape)
    return shape, x, f


def test_conv_golden_every_algorithm(tk, oracle):
    g = np.load(os.path.join(GOLDEN, "conv.npz"))
    tiled = ["tiled_t4x5_v4x2", "tiled_t1x1_v1x1", "tiled_t2x2_v2x8", "tiled_t3x1_v8x4"]
    for i, s in enumerate(json.loads(str(g["meta"]))):
        shape, x, f = conv_case(tk, oracle, s)
        want = g[f"naive{i}"]
        for p in ["naive", "im2col", tiled[i % len(tiled)]]:
            got = tk.conv2d(x, f, shape, tk.parse_conv_params(p))
            assert same(got, want), (s, p)
        assert same(tk.im2col(x, shape), g[f"im2col{i}"]), s
        for m in (2, 4):
            key = f"wino{m}_{i}"
            if key in g.files:
                out, mults, tiles = tk.conv2d_winograd(x, f, shape, tk.ConvAlgoParams("winograd", m, m))
                assert same(out, g[key]), (s, m)       # Winograd FP32 is bit-identical too
                assert [mults, tiles] == s[f"wino{m}_stats"]


def test_conv_im2col_with_explicit_configs(tk, oracle):
    s = tk.ConvShape(2, 12, 10, 6, 8, 3, 3, 2, True)
    O = oracle
    conv = O.Conv(2, 12, 10, 6, 8, 3, 3, 2, True)
    x = O.fill_random(int(np.prod(conv.in_shape)), 81).reshape(conv.in_shape)
    f = O.fill_random(int(np.prod(conv.filt_shape)), 82).reshape(conv.filt_shape)
    want = O.conv2d_naive(conv, x, f)
    b200 = tk.b200_device()
    for name in STOCK + ["8x8_16x16_loc_db", "4x8_32x8_loc_db"]:
        got = tk.conv2d_im2col(x, f, s, tk.parse_gemm_config(name), b200)
        assert same(got, want), name


def test_filter_matrix(tk, oracle):
    f = oracle.fill_random(3 * 3 * 5 * 7, 3).reshape(3, 3, 5, 7)
    assert same(tk.filter_matrix(f), oracle.filter_matrix(f))


def test_batch_independence(tk, oracle):
    """test_conv.cpp:268-293: image n of a batch equals the single-image run."""
    s1 = tk.ConvShape(1, 7, 7, 4, 3, 3, 3, 1, True)
    s2 = tk.ConvShape(2, 7, 7, 4, 3, 3, 3, 1, True)
    a = oracle.fill_random(7 * 7 * 4, 91).reshape(1, 7, 7, 4)
    b = oracle.fill_random(7 * 7 * 4, 92).reshape(1, 7, 7, 4)
    f = oracle.fill_random(3 * 3 * 4 * 3, 93).reshape(3, 3, 4, 3)
    both = np.concatenate([a, b])
    for p in ["naive", "im2col", "tiled_t2x2_v2x2", "winograd_t2x2", "winograd_t4x4"]:
        pp = tk.parse_conv_params(p)
        ob = tk.conv2d(both, f, s2, pp)
        assert same(ob[0], tk.conv2d(a, f, s1, pp)[0]) and same(ob[1], tk.conv2d(b, f, s1, pp)[0]), p


VGG = [  # (name, H, C, K) -- proj/data/vgg_layers.csv
    ("vgg_conv1_1", 224, 3, 64), ("vgg_conv1_2", 224, 64, 64), ("vgg_conv2_1", 112, 64, 128),
    ("vgg_conv2_2", 112, 128, 128), ("vgg_conv3_1", 56, 128, 256), ("vgg_conv3_2", 56, 256, 256),
    ("vgg_conv4_1", 28, 256, 512), ("vgg_conv4_2", 28, 512, 512), ("vgg_conv5", 14, 512, 512),
]


@pytest.mark.parametrize("name,H,C,K", VGG)
def test_vgg_layers_batch1_exact(tk, oracle, name, H, C, K):
    """Every VGG-16 layer shape at batch 1, exact FP32 vs the oracle."""
    import torch
    s = tk.ConvShape(1, H, H, C, K, 3, 3, 1, True)
    conv = oracle.Conv(1, H, H, C, K, 3, 3, 1, True)
    x = oracle.fill_random(int(np.prod(conv.in_shape)), 5).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), 6).reshape(conv.filt_shape)
    want = oracle.conv2d_naive(conv, x, f)
    dx, df = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
    dy = torch.empty(conv.out_shape, device="cuda")
    tk.conv2d_dev(dx, df, dy, s, tk.parse_conv_params("im2col"))
    assert same(dy.cpu().numpy(), want)


# ---- runtime register tiles (microkernel_generic, gemm.hpp:247-292) -------
GENERIC = ["3x5_8x8_loc", "5x3_4x16_noloc", "7x1_16x16_loc_db", "1x7_16x8_loc", "6x6_8x8_loc_db",
           "12x12_8x8_loc", "3x20_8x4_loc", "16x8_8x8_loc", "9x2_8x16_noloc"]


@pytest.mark.parametrize("cfg", GENERIC)
def test_gemm_tiled_generic_register_tiles(tk, oracle, cfg):
    """Configs outside h, w in {1, 2, 4, 8} run bit-exact (the reference's
    generic microkernel) instead of raising; all op combos, ragged tails,
    alpha/beta."""
    dev = tk.b200_device()
    ok, msg = tk.validate_config(tk.parse_gemm_config(cfg), dev)
    assert ok, msg
    for (m, n, k) in [(67, 45, 17), (128, 96, 64), (33, 1, 130)]:
        for ta in (0, 1):
            for tb in (0, 1):
                a = oracle.fill_random(m * k, 1)
                b = oracle.fill_random(k * n, 2)
                c = oracle.fill_random(m * n, 3)
                want = oracle.gemm_naive(m, n, k, 1.5, -0.5, ta, tb, a, b, c)
                shape = tk.GemmShape(m, n, k, 1.5, -0.5, "t" if ta else "n", "t" if tb else "n")
                got = tk.gemm_tiled(a, b, c, shape, tk.parse_gemm_config(cfg), dev)
                assert same(got, want), (cfg, m, n, k, ta, tb)


@pytest.mark.parametrize("params", ["tiled_t4x5_v4x2", "tiled_t1x1_v1x1", "tiled_t3x7_v2x8",
                                    "tiled_t8x8_v8x1", "tiled_t5x5_v1x4", "tiled_t2x3_v8x8",
                                    "tiled_t4x4_v4x4"])
@pytest.mark.parametrize("shape", [(2, 13, 11, 8, 20, 3, 1, True), (1, 15, 15, 3, 64, 3, 1, True),
                                   (2, 16, 14, 12, 10, 3, 2, True), (1, 9, 12, 6, 7, 3, 1, False),
                                   (1, 20, 20, 3, 64, 7, 2, True), (3, 7, 7, 32, 48, 1, 1, True)])
def test_conv2d_tiled_patch_geometry_bit_exact(tk, oracle, params, shape):
    """conv2d_tiled's tile_rows x tile_cols patch, feature_vector and
    channel_vector shape the CTA (2-D pixel patches per thread, channel
    groups per staging copy); outputs stay bit-identical to conv2d_naive."""
    n, h, w, c, k, r, st, same_pad = shape
    s = tk.ConvShape(n, h, w, c, k, r, r, st, same_pad)
    conv = oracle.Conv(n, h, w, c, k, r, r, st, same_pad)
    x = oracle.fill_random(int(np.prod(conv.in_shape)), 5).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), 6).reshape(conv.filt_shape)
    want = oracle.conv2d_naive(conv, x, f)
    got = tk.conv2d(x, f, s, tk.parse_conv_params(params))
    assert same(got, want), (params, shape)


def test_conv2d_im2col_with_generic_config(tk, oracle):
    """conv2d_im2col(cfg, dev) honours an explicit non-power-of-two config."""
    s = tk.ConvShape(2, 10, 9, 5, 7, 3, 3, 1, True)
    conv = oracle.Conv(2, 10, 9, 5, 7, 3, 3, 1, True)
    x = oracle.fill_random(int(np.prod(conv.in_shape)), 8).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), 9).reshape(conv.filt_shape)
    want = oracle.conv2d_naive(conv, x, f)
    for cfg in ("3x5_8x8_loc", "5x3_4x16_noloc"):
        got = tk.conv2d_im2col(x, f, s, tk.parse_gemm_config(cfg), tk.b200_device())
        assert same(got, want), cfg
