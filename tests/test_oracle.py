"""CPU: pin the oracle (oracle/tk_oracle.c) before trusting it.

1. Known answers from the reference's own unit tests (test_gemm.cpp,
   test_conv.cpp, test_winograd.cpp, acceptance.cpp criterion 5).
2. Golden fixtures produced by the UNMODIFIED reference headers
   (tests/golden/make_golden.py) -- bit-exact.
3. When oracle/_ref is built (this container), live cross-checks against the
   reference on fresh random shapes.
"""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


# ---------------------------------------------------------------- known answers

def test_fill_random_matches_golden(oracle):
    g = np.load(os.path.join(GOLDEN, "rng.npz"))
    for seed, values in zip(g["seeds"], g["values"]):
        assert np.array_equal(bits(oracle.fill_random(256, int(seed))), bits(values))


def test_gemm_known_answers(oracle):
    # test_gemm.cpp:199-233
    a = np.array([1, 0, 0, 1], np.float32)
    b = np.array([5, 6, 7, 8], np.float32)
    assert np.array_equal(oracle.gemm_naive(2, 2, 2, 1, 0, 0, 0, a, b, None), b)
    a = np.array([1, 3, 2, 4], np.float32)          # [[1,2],[3,4]] column-major
    b = np.array([5, 7, 6, 8], np.float32)
    out = oracle.gemm_naive(2, 2, 2, 1, 0, 0, 0, a, b, None)
    assert out.tolist() == [19, 43, 22, 50]
    out = oracle.gemm_naive(1, 1, 1, 1, 0, 0, 0, np.array([2], np.float32),
                            np.array([3], np.float32), np.array([np.nan], np.float32))
    assert out[0] == 6.0                              # beta == 0: C never read
    c = oracle.fill_random(16, 3)
    out = oracle.gemm_naive(4, 4, 4, 0, 1, 0, 0, oracle.fill_random(16, 1),
                            oracle.fill_random(16, 2), c)
    assert np.array_equal(bits(out), bits(c))         # alpha 0, beta 1


def test_conv_known_answers(oracle):
    O = oracle
    ones = lambda *s: np.ones(s, np.float32)  # noqa: E731
    out = O.conv2d_naive(O.Conv(1, 4, 4, 1, 1, 3, 3, 1, False), ones(1, 4, 4, 1), ones(3, 3, 1, 1))
    assert out.shape == (1, 2, 2, 1) and np.all(out == 9)
    out = O.conv2d_naive(O.Conv(1, 3, 3, 1, 1, 3, 3, 1, True), ones(1, 3, 3, 1), ones(3, 3, 1, 1))
    assert out[0, :, :, 0].tolist() == [[4, 6, 4], [6, 9, 6], [4, 6, 4]]
    out = O.conv2d_naive(O.Conv(1, 3, 3, 4, 2, 3, 3, 1, False), ones(1, 3, 3, 4), ones(3, 3, 4, 2))
    assert out.ravel().tolist() == [36, 36]
    x = np.arange(25, dtype=np.float32).reshape(1, 5, 5, 1)
    out = O.conv2d_naive(O.Conv(1, 5, 5, 1, 1, 1, 1, 2, False), x, ones(1, 1, 1, 1))
    assert out[0, :, :, 0][0, 0] == 0 and out[0, 0, 1, 0] == 2 and out[0, 1, 0, 0] == 10
    assert out[0, 2, 2, 0] == 24


def test_same_padding_is_tf_style(oracle):
    # ResNet stem 7x7/s2 on 224 -> 112: pad_top = pad_left = 2 (config.hpp:148-181)
    s = oracle.Conv(1, 224, 224, 3, 64, 7, 7, 2, True)
    assert (s.out_rows, s.pad_top, s.pad_left) == (112, 2, 2)


def test_im2col_known_answers(oracle):
    O = oracle
    s = O.Conv(1, 3, 3, 1, 1, 2, 2, 1, False)        # test_conv.cpp:207-228
    x = np.arange(1, 10, dtype=np.float32).reshape(1, 3, 3, 1)
    p = O.im2col(s, x).reshape(4, 4, order="F")
    assert p[0].tolist() == [1, 2, 4, 5]
    assert int((p == 5).sum()) == 4
    s = O.Conv(1, 2, 2, 1, 1, 3, 3, 1, True)          # test_conv.cpp:230-243
    p = O.im2col(s, np.array([1, 2, 3, 4], np.float32).reshape(1, 2, 2, 1)).reshape(4, 9, order="F")
    assert p[0, 0] == 0 and p[0, 4] == 1 and p[0, 5] == 2 and p[0, 7] == 3 and p[0, 8] == 4


def test_winograd_known_answers(oracle):
    O = oracle
    bt, g, at = O.winograd_plan(2)
    assert bt.shape == (4, 4) and g.shape == (4, 3) and at.shape == (2, 4)
    bt, g, at = O.winograd_plan(4)
    assert bt.shape == (6, 6) and g.shape == (6, 3) and at.shape == (4, 6)
    with pytest.raises(ValueError):
        O.winograd_plan(3)
    # multiply counts on 8x8x1 (test_winograd.cpp:158-178; acceptance 5)
    s = O.Conv(1, 8, 8, 1, 1, 3, 3, 1, True)
    x = O.fill_random(64, 1).reshape(1, 8, 8, 1)
    f = O.fill_random(9, 2).reshape(3, 3, 1, 1)
    _, m2, t2 = O.conv2d_winograd(s, 2, x, f)
    _, m4, t4 = O.conv2d_winograd(s, 4, x, f)
    assert (m2, t2, m4, t4) == (256, 16, 144, 4)
    # central tap = identity (test_winograd.cpp:73-90)
    f = np.zeros((3, 3, 1, 1), np.float32)
    f[1, 1] = 1
    for m in (2, 4):
        out, _, _ = O.conv2d_winograd(s, m, x, f)
        assert O.max_scaled_error(out, x) <= 1e-5


# ---------------------------------------------------------------- golden fixtures

def test_gemm_golden_bit_exact(oracle):
    g = np.load(os.path.join(GOLDEN, "gemm.npz"))
    for i, c in enumerate(json.loads(str(g["meta"]))):
        m, n, k = c["m"], c["n"], c["k"]
        a = oracle.fill_random(m * k, c["seed"])
        b = oracle.fill_random(k * n, c["seed"] + 1)
        cc = oracle.fill_random(m * n, c["seed"] + 2)
        out = oracle.gemm_naive(m, n, k, c["alpha"], c["beta"], c["ta"], c["tb"], a, b, cc)
        assert np.array_equal(bits(out), bits(g[f"out{i}"])), c


def conv_case(oracle, s):
    conv = oracle.Conv(s["batch"], s["in_rows"], s["in_cols"], s["channels"], s["features"],
                       s["window"], s["window"], s["stride"], s["same"])
    x = oracle.fill_random(int(np.prod(conv.in_shape)), s["seed"]).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), s["seed"] + 1).reshape(conv.filt_shape)
    return conv, x, f


def test_conv_golden_bit_exact(oracle):
    g = np.load(os.path.join(GOLDEN, "conv.npz"))
    nwino = 0
    for i, s in enumerate(json.loads(str(g["meta"]))):
        conv, x, f = conv_case(oracle, s)
        assert np.array_equal(bits(oracle.conv2d_naive(conv, x, f)), bits(g[f"naive{i}"])), s
        assert np.array_equal(bits(oracle.im2col(conv, x)), bits(g[f"im2col{i}"])), s
        for m in (2, 4):
            key = f"wino{m}_{i}"
            if key in g.files:
                out, mults, tiles = oracle.conv2d_winograd(conv, m, x, f)
                assert np.array_equal(bits(out), bits(g[key])), (s, m)
                assert [mults, tiles] == s[f"wino{m}_stats"]
                nwino += 1
    assert nwino >= 10


# ---------------------------------------------------------------- live reference

needs_ref = pytest.mark.skipif(
    not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libtkref.so")),
    reason="oracle/_ref not built")


@needs_ref
def test_live_reference_cross_check(oracle):
    rng = np.random.default_rng(7)
    for trial in range(12):
        m, n, k = (int(v) for v in rng.integers(1, 90, 3))
        ta, tb = (int(v) for v in rng.integers(0, 2, 2))
        a = oracle.fill_random(m * k, trial)
        b = oracle.fill_random(k * n, trial + 100)
        c = oracle.fill_random(m * n, trial + 200)
        want = oracle.ref_gemm_tiled(m, n, k, 0.75, -1.25, ta, tb, a, b, c, "8x4_8x16_loc_db")
        got = oracle.gemm_naive(m, n, k, 0.75, -1.25, ta, tb, a, b, c)
        assert np.array_equal(bits(got), bits(want))
    for trial in range(8):
        s = oracle.Conv(int(rng.integers(1, 3)), int(rng.integers(5, 16)), int(rng.integers(5, 16)),
                        int(rng.choice([3, 4, 16])), int(rng.choice([5, 8])), 3, 3,
                        int(rng.integers(1, 3)), bool(rng.integers(0, 2)))
        x = oracle.fill_random(int(np.prod(s.in_shape)), trial).reshape(s.in_shape)
        f = oracle.fill_random(int(np.prod(s.filt_shape)), trial + 1).reshape(s.filt_shape)
        want = oracle.ref_conv2d(s, "tiled_t4x5_v4x2", x, f)
        assert np.array_equal(bits(oracle.conv2d_naive(s, x, f)), bits(want))
        if s.stride == 1:
            w, _, _ = oracle.ref_conv2d_winograd(s, 4, x, f)
            o, _, _ = oracle.conv2d_winograd(s, 4, x, f)
            assert np.array_equal(bits(o), bits(w))
