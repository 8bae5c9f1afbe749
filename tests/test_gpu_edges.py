"""Edge cases across every arithmetic path: empty and degenerate shapes,
single-pixel planes, ragged channel/feature counts, misaligned device
buffers.  Each either matches the oracle (bit-exact for FP32, the stated
tolerance for TF32/BF16) or fails with the reference's exception class --
never a crash, a hang or silent garbage."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"tf32": 1e-3, "bf16": 5e-3}
PRECS = ["fp32", "tf32", "bf16"]


def _gemm(tk, oracle, m, n, k, prec, alpha=1.5, beta=-0.5):
    a = oracle.fill_random(m * k, 1)
    b = oracle.fill_random(k * n, 2)
    c = oracle.fill_random(m * n, 3)
    want = oracle.gemm_naive(m, n, k, alpha, beta, 0, 0, a, b, c)
    shape = tk.GemmShape(m, n, k, alpha, beta)
    if prec == "fp32":
        got = tk.gemm_tiled(a, b, c, shape, tk.parse_gemm_config("4x4_8x8_loc"), tk.b200_device())
    else:
        import torch
        da, db, dc = (torch.from_numpy(v).cuda() for v in (a, b, c))
        out = torch.full((m * n,), float("nan"), device="cuda")
        tk.gemm_dev(da, db, dc, out, shape, precision=prec)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
    return np.asarray(got).reshape(-1), want


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("m,n,k", [(0, 5, 3), (4, 0, 3), (4, 5, 0)])
def test_gemm_zero_dimension_is_a_shape_error(tk, oracle, m, n, k, prec):
    """The reference's Matrix rejects a zero dimension (tensor.hpp:21-26):
    ShapeError on every path, before any launch."""
    with pytest.raises(tk.ShapeError, match="positive"):
        _gemm(tk, oracle, m, n, k, prec)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (1, 300, 1), (300, 1, 2), (2, 3, 700)])
def test_gemm_thin_shapes(tk, oracle, m, n, k, prec):
    got, want = _gemm(tk, oracle, m, n, k, prec)
    if prec == "fp32":
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    else:
        assert oracle.max_scaled_error(got, want) <= TOL[prec]


def _conv(tk, oracle, N, H, W, C, K, R, stride, same, prec, algo="im2col"):
    s = tk.ConvShape(N, H, W, C, K, R, R, stride, same)
    conv = oracle.Conv(N, H, W, C, K, R, R, stride, same)
    x = oracle.fill_random(max(1, int(np.prod(conv.in_shape))), 4)[: int(np.prod(conv.in_shape))]
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), 5)
    x = x.reshape(conv.in_shape)
    f = f.reshape(conv.filt_shape)
    want = oracle.conv2d_naive(conv, x, f)
    got = tk.conv2d(x, f, s, tk.parse_conv_params(algo), precision=prec)
    return np.asarray(got), want


@pytest.mark.parametrize("prec", PRECS)
def test_conv_empty_batch_is_a_shape_error(tk, oracle, prec):
    """Tensor4 rejects a zero dimension in the reference (tensor.hpp:96-99)."""
    with pytest.raises(tk.ShapeError, match="positive"):
        _conv(tk, oracle, 0, 8, 8, 32, 64, 3, 1, True, prec)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("shape", [(2, 1, 1, 32, 64, 3, 1, True),    # one pixel: centre tap only
                                   (1, 2, 2, 64, 128, 3, 1, True),
                                   (3, 5, 3, 32, 32, 1, 2, True),    # 1x1/s2 on an odd plane
                                   (1, 3, 3, 32, 64, 3, 1, False)])  # Valid: one output pixel
def test_conv_tiny_planes(tk, oracle, shape, prec):
    got, want = _conv(tk, oracle, *shape, prec)
    if prec == "fp32":
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    else:
        assert oracle.max_scaled_error(got, want) <= TOL[prec]


@pytest.mark.parametrize("C,K", [(5, 8), (7, 12), (33, 20), (3, 4)])
def test_conv_ragged_channels_tensor_cores(tk, oracle, C, K):
    """Channel counts that are no whole slab go through the gather path."""
    got, want = _conv(tk, oracle, 2, 9, 11, C, K, 3, 1, True, "tf32")
    assert oracle.max_scaled_error(got, want) <= TOL["tf32"]


@pytest.mark.parametrize("K", [5, 7, 30])
def test_conv_ragged_features(tk, oracle, K):
    """Exact FP32 takes any feature count; the tensor-core path needs whole
    16-byte output rows and says so with CapabilityError."""
    got, want = _conv(tk, oracle, 1, 6, 6, 8, K, 3, 1, True, "fp32")
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    if K % 4:
        with pytest.raises(tk.CapabilityError):
            _conv(tk, oracle, 1, 6, 6, 8, K, 3, 1, True, "tf32")


def test_misaligned_device_buffers(tk, oracle):
    """Device pointers off the 16-byte grid: the tensor-core path either
    computes the right answer or raises CapabilityError, never faults."""
    import torch
    s = tk.ConvShape(1, 8, 8, 32, 64, 3, 3, 1, True)
    conv = oracle.Conv(1, 8, 8, 32, 64, 3, 3, 1, True)
    x = oracle.fill_random(int(np.prod(conv.in_shape)), 6).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), 7).reshape(conv.filt_shape)
    want = oracle.conv2d_naive(conv, x, f)
    bx = torch.zeros(x.size + 1, device="cuda")
    bx[1:] = torch.from_numpy(x.reshape(-1)).cuda()
    dx = bx[1:].view(conv.in_shape)
    df = torch.from_numpy(f).cuda()
    dy = torch.full(conv.out_shape, float("nan"), device="cuda")
    for prec in ("fp32", "tf32"):
        try:
            tk.conv2d_dev(dx, df, dy, s, tk.parse_conv_params("im2col"), precision=prec)
            torch.cuda.synchronize()
        except tk.CapabilityError:
            continue
        got = dy.cpu().numpy()
        if prec == "fp32":
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
        else:
            assert oracle.max_scaled_error(got, want) <= TOL[prec]
