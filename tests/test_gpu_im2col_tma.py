"""GPU parity of the im2col-mode TMA convolution path (tk_exec_options.tc_mode
= TK_TC_IM2COL): output pixels on the MMA M side, loaded 128 at a time in
NHW order by cp.async.bulk.tensor.*.im2col, one filter tap per K-slab.

Checked against the CPU oracle's conv2d_naive (conv.hpp:74-113) with the
tolerances of test_gpu_tc.py (TF32 <= 1e-3, BF16 <= 5e-3 max_scaled_error,
numeric.hpp:39-56); runs are deterministic bit for bit.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"tf32": 1e-3, "bf16": 5e-3}


def run_mode(tk, x, f, shape, prec, mode="im2col", split=0):
    import torch
    dx, df = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
    dy = torch.full(shape.out_shape, float("nan"), device="cuda")
    opts = tk.exec_options(prec, mode=mode, split=split)
    p = tk.parse_conv_params("im2col")
    ws = torch.empty(max(tk.conv2d_workspace_size(shape, p, options=opts), 4) // 4 + 1,
                     device="cuda")
    tk.conv2d_dev(dx, df, dy, shape, p, workspace=ws, options=opts)
    torch.cuda.synchronize()
    return dy.cpu().numpy()


def case(oracle, N, H, W, C, K, R, stride, same, seed=11):
    conv = oracle.Conv(N, H, W, C, K, R, R, stride, same)
    x = oracle.fill_random(int(np.prod(conv.in_shape)), seed).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), seed + 1).reshape(conv.filt_shape)
    return conv, x, f, oracle.conv2d_naive(conv, x, f)


SHAPES = [
    # N, H, W, C, K, R, stride, same
    (2, 14, 14, 64, 256, 3, 1, True),     # 14x14 planes: tiles cross image boundaries
    (3, 7, 7, 128, 128, 3, 1, True),      # 7x7 planes (ResNet res5 geometry)
    (1, 28, 28, 32, 128, 3, 1, True),
    (2, 17, 23, 32, 96, 3, 1, True),      # ragged plane, features not a multiple of 32
    (2, 20, 18, 32, 64, 3, 1, False),     # Valid
    (2, 20, 18, 64, 64, 3, 2, True),      # stride 2, Same (pad smaller first)
    (2, 21, 19, 32, 128, 3, 2, False),    # stride 2, Valid, odd plane
    (2, 16, 16, 64, 128, 1, 1, True),     # 1x1
    (2, 15, 15, 64, 128, 1, 2, True),     # 1x1 stride 2
    (2, 12, 12, 64, 64, 5, 1, True),      # 5x5
    (1, 20, 20, 64, 64, 7, 2, True),      # 7x7 / 2
    (1, 4, 4, 64, 32, 3, 1, True),        # tiny tensor (< 128 KiB descriptor workaround)
    (1, 1, 1, 64, 64, 3, 1, True),        # one-pixel plane
]


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
@pytest.mark.parametrize("shape", SHAPES)
def test_im2col_tma_matches_oracle(tk, oracle, shape, prec):
    N, H, W, C, K, R, stride, same = shape
    if prec == "bf16" and C % 64:
        pytest.skip("BF16 slabs hold 64 channels")
    conv, x, f, want = case(oracle, *shape)
    s = tk.ConvShape(N, H, W, C, K, R, R, stride, same)
    got = run_mode(tk, x, f, s, prec)
    assert not np.isnan(got).any()
    err = oracle.max_scaled_error(got, want)
    assert err <= TOL[prec], err


@pytest.mark.parametrize("split", [1, 3])
def test_im2col_tma_split_k_and_determinism(tk, oracle, split):
    shape = (4, 14, 14, 128, 256, 3, 1, True)
    conv, x, f, want = case(oracle, *shape, seed=21)
    s = tk.ConvShape(*shape[:5], 3, 3, 1, True)
    a = run_mode(tk, x, f, s, "tf32", split=split)
    b = run_mode(tk, x, f, s, "tf32", split=split)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert oracle.max_scaled_error(a, want) <= TOL["tf32"]


def test_im2col_tma_matches_box_path(tk, oracle):
    """Same convolution through the tiled-box path and the im2col path."""
    shape = (4, 28, 28, 128, 128, 3, 1, True)
    conv, x, f, want = case(oracle, *shape, seed=31)
    s = tk.ConvShape(*shape[:5], 3, 3, 1, True)
    a = run_mode(tk, x, f, s, "tf32", mode="im2col")
    b = run_mode(tk, x, f, s, "tf32", mode="auto")
    assert oracle.max_scaled_error(a, want) <= TOL["tf32"]
    assert oracle.max_scaled_error(b, want) <= TOL["tf32"]
    # both truncate the same TF32 operands: differences are summation order only
    assert oracle.max_scaled_error(a, b) <= 2e-5


def test_im2col_mode_rejects_unboxable_channels(tk, oracle):
    import torch
    # (C <= 4 runs as narrow-pixel im2col; 5 channels are neither a slab
    # nor a 16-byte pixel)
    s = tk.ConvShape(1, 8, 8, 5, 16, 3, 3, 1, True)
    opts = tk.exec_options("tf32", mode="im2col")
    with pytest.raises(tk.CapabilityError):
        tk.conv2d_workspace_size(s, tk.parse_conv_params("im2col"), options=opts)


# Gather mode (channel counts that are not whole slabs: VGG conv1_1, the
# ResNet stem): producer warps stage the input rows of each 128-pixel run in
# shared memory and build the K-slabs from there.
GATHER_SHAPES = [
    # N, H, W, C, K, R, stride, same
    (2, 224, 224, 3, 64, 3, 1, True),    # conv1_1 geometry (runs cross rows)
    (2, 224, 224, 3, 64, 7, 2, True),    # ResNet stem
    (3, 13, 13, 3, 16, 3, 1, True),      # a run spans ~10 rows and 3 images
    (1, 129, 127, 5, 32, 3, 1, False),   # Valid, ragged rows
    (2, 40, 33, 7, 48, 5, 2, True),      # stride 2, 5x5
    (1, 1, 1, 3, 16, 3, 1, True),        # one pixel
]


@pytest.mark.parametrize("shape", GATHER_SHAPES)
def test_gather_mode_matches_oracle(tk, oracle, shape):
    N, H, W, C, K, R, stride, same = shape
    conv, x, f, want = case(oracle, *shape, seed=41)
    s = tk.ConvShape(N, H, W, C, K, R, R, stride, same)
    got = run_mode(tk, x, f, s, "tf32", mode="gather")
    assert not np.isnan(got).any()
    assert oracle.max_scaled_error(got, want) <= TOL["tf32"]


# Automatic operand-path rules (plan_conv): each shape lands on a different
# path in BF16 / TF32; all must agree with the oracle.
AUTO_SHAPES = [
    # N, H, W, C, K, R, stride, same       path (bf16 / tf32)
    (2, 16, 16, 64, 128, 1, 1, True),      # im2col (K >= 2C) / pointwise
    (2, 16, 16, 128, 128, 1, 1, True),     # one-tap halo / pointwise
    (4, 7, 7, 256, 128, 1, 1, True),       # im2col (7 x 7) / pointwise
    (2, 28, 28, 128, 256, 3, 1, True),     # im2col (wide 3x3, plane >= 28) / im2col
    (2, 28, 28, 64, 128, 3, 1, True),      # halo (128-wide tiles)
    (2, 30, 30, 256, 128, 1, 2, True),     # strided 1x1: compacting GEMM / im2col
]


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
@pytest.mark.parametrize("shape", AUTO_SHAPES)
def test_auto_paths_match_oracle(tk, oracle, shape, prec):
    N, H, W, C, K, R, stride, same = shape
    conv, x, f, want = case(oracle, *shape, seed=51)
    s = tk.ConvShape(N, H, W, C, K, R, R, stride, same)
    got = run_mode(tk, x, f, s, prec, mode="auto")
    assert not np.isnan(got).any()
    assert oracle.max_scaled_error(got, want) <= TOL[prec]
