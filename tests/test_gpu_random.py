"""Randomised convolution parity in the spirit of the reference's acceptance
criterion 3 (acceptance.cpp:163-233: random shapes, seed 42): every operand
path the tensor-core planner can pick (halo, pixel boxes incl. flat-row and
multi-image tiles, traversal-stride boxes, pointwise GEMM, gather, split-K
and wave tails) and the exact path, on seeded random shapes.  FP32 exact is
bit-identical; TF32 / BF16 / 3xTF32 within their stated bars."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"tf32": 1e-3, "bf16": 5e-3, "3xtf32": 5e-5}


def random_shapes(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        r = int(rng.choice([1, 3, 3, 3, 5, 7]))
        stride = int(rng.choice([1, 1, 2]))
        same = bool(rng.random() < 0.75)
        h = int(rng.integers(max(1, r if not same else 1), 40))
        w = int(rng.integers(max(1, r if not same else 1), 40))
        c = int(rng.choice([1, 3, 5, 16, 32, 64, 96, 128, 192, 256]))
        k = int(rng.choice([4, 8, 12, 32, 64, 96, 128, 256, 512]))
        n = int(rng.integers(1, 6))
        if not same and (h < r or w < r):
            continue
        if n * h * w * c * k * r * r > 120e6:  # keep the CPU oracle in seconds
            continue
        out.append((n, h, w, c, k, r, stride, same))
    return out


SHAPES = random_shapes(42, 40)


def run(tk, oracle, shape, prec, seed):
    import torch
    n, h, w, c, k, r, stride, same = shape
    s = tk.ConvShape(n, h, w, c, k, r, r, stride, same)
    conv = oracle.Conv(n, h, w, c, k, r, r, stride, same)
    x = oracle.fill_random(int(np.prod(conv.in_shape)), seed).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), seed + 1).reshape(conv.filt_shape)
    want = oracle.conv2d_naive(conv, x, f)
    dx, df = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
    dy = torch.full(conv.out_shape, float("nan"), device="cuda")
    tk.conv2d_dev(dx, df, dy, s, tk.parse_conv_params("im2col"), precision=prec)
    torch.cuda.synchronize()
    return dy.cpu().numpy(), want


@pytest.mark.parametrize("i", range(len(SHAPES)), ids=[str(s) for s in SHAPES])
def test_random_exact_bit_identical(tk, oracle, i):
    got, want = run(tk, oracle, SHAPES[i], "fp32", 100 + i)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("prec", ["tf32", "bf16", "3xtf32"])
@pytest.mark.parametrize("i", range(len(SHAPES)), ids=[str(s) for s in SHAPES])
def test_random_tensor_cores(tk, oracle, i, prec):
    shape = SHAPES[i]
    try:
        got, want = run(tk, oracle, shape, prec, 200 + i)
    except tk.CapabilityError:
        # the documented limit: output features must fill 16-byte rows
        assert shape[4] % 4 != 0
        return
    assert not np.isnan(got).any()
    assert oracle.max_scaled_error(got, want) <= TOL[prec]


def random_gemms(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m, n, k = (int(v) for v in rng.integers(1, 700, 3))
        ta, tb = (int(v) for v in rng.integers(0, 2, 2))
        alpha = float(rng.choice([1.0, 0.5, -1.25]))
        beta = float(rng.choice([0.0, 1.0, -0.5]))
        out.append((m, n, k, ta, tb, alpha, beta))
    return out


GEMMS = random_gemms(20240811, 30)  # acceptance.cpp:103-157's seed


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16", "3xtf32"])
@pytest.mark.parametrize("i", range(len(GEMMS)), ids=[str(g) for g in GEMMS])
def test_random_gemm(tk, oracle, i, prec):
    import torch
    m, n, k, ta, tb, alpha, beta = GEMMS[i]
    a = oracle.fill_random(m * k, 300 + i)
    b = oracle.fill_random(k * n, 400 + i)
    c = oracle.fill_random(m * n, 500 + i)
    want = oracle.gemm_naive(m, n, k, alpha, beta, ta, tb, a, b, c)
    da, db, dc = (torch.from_numpy(v).cuda() for v in (a, b, c))
    out = torch.full((m * n,), float("nan"), device="cuda")
    shape = tk.GemmShape(m, n, k, alpha, beta, "t" if ta else "n", "t" if tb else "n")
    if prec == "fp32":
        tk.gemm_dev(da, db, dc, out, shape, tk.parse_gemm_config("8x4_8x16_loc"), precision="fp32")
    else:
        tk.gemm_dev(da, db, dc, out, shape, precision=prec)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    if prec == "fp32":
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    else:
        assert oracle.max_scaled_error(got, want) <= TOL[prec]
