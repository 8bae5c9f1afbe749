"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads ``oracle/_build/libtkoracle.so`` (the C restatement, tk_oracle.c) and,
when present, ``oracle/_ref/libtkref.so`` (the unmodified reference headers
behind ref_shim.cpp).  Only tests/, ``__graft_entry__.smoke()`` and the CPU
legs of bench.py import this module; the product path never does.

Arrays follow the reference conventions: column-major matrices passed as
flat float32 vectors (``Matrix::data``), NHWC / HWCK tensors as C-contiguous
float32 arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libtkoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtkref.so")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


class ConvShapeC(C.Structure):
    """Mirror of tko_conv_shape / ref_shim ShapeC (reference ConvShape)."""

    _fields_ = [
        ("batch", C.c_size_t),
        ("in_rows", C.c_size_t),
        ("in_cols", C.c_size_t),
        ("channels", C.c_size_t),
        ("features", C.c_size_t),
        ("window_rows", C.c_size_t),
        ("window_cols", C.c_size_t),
        ("stride", C.c_size_t),
        ("same", C.c_int),
    ]


@dataclass(frozen=True)
class Conv:
    """Python twin of tilekit::ConvShape (reference config.hpp:137-195)."""

    batch: int
    in_rows: int
    in_cols: int
    channels: int
    features: int
    window_rows: int
    window_cols: int
    stride: int = 1
    same: bool = True

    def c(self) -> ConvShapeC:
        return ConvShapeC(self.batch, self.in_rows, self.in_cols, self.channels,
                          self.features, self.window_rows, self.window_cols,
                          self.stride, 1 if self.same else 0)

    def _out(self, n: int, w: int) -> int:
        if not self.same:
            return 0 if n < w else (n - w) // self.stride + 1
        return (n + self.stride - 1) // self.stride

    @property
    def out_rows(self) -> int:
        return self._out(self.in_rows, self.window_rows)

    @property
    def out_cols(self) -> int:
        return self._out(self.in_cols, self.window_cols)

    def _pad(self, n: int, w: int) -> int:
        if not self.same:
            return 0
        out = self._out(n, w)
        span = (out - 1) * self.stride + w if out > 0 else w
        return (span - n) // 2 if span > n else 0

    @property
    def pad_top(self) -> int:
        return self._pad(self.in_rows, self.window_rows)

    @property
    def pad_left(self) -> int:
        return self._pad(self.in_cols, self.window_cols)

    @property
    def in_shape(self):
        return (self.batch, self.in_rows, self.in_cols, self.channels)

    @property
    def filt_shape(self):
        return (self.window_rows, self.window_cols, self.channels, self.features)

    @property
    def out_shape(self):
        return (self.batch, self.out_rows, self.out_cols, self.features)

    def flops(self) -> int:
        return (2 * self.batch * self.out_rows * self.out_cols * self.features *
                self.window_rows * self.window_cols * self.channels)

    def key(self) -> str:
        return (f"conv_n{self.batch}_{self.in_rows}x{self.in_cols}x{self.channels}"
                f"_k{self.features}_f{self.window_rows}x{self.window_cols}"
                f"_s{self.stride}_{'same' if self.same else 'valid'}")


_lib = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.tko_fill_random.argtypes = [_f32p, C.c_size_t, C.c_uint64]
        L.tko_fnv1a.argtypes = [C.c_char_p]
        L.tko_fnv1a.restype = C.c_uint64
        L.tko_gemm_naive.argtypes = [C.c_size_t] * 3 + [C.c_float] * 2 + [C.c_int] * 2 + [_f32p] * 4
        L.tko_gemm_batched_strided.argtypes = [_f32p, C.c_size_t, _f32p, C.c_size_t, _f32p,
                                               C.c_size_t] + [C.c_size_t] * 4
        L.tko_gemm_batched_strided.restype = C.c_uint64
        L.tko_conv2d_naive.argtypes = [C.POINTER(ConvShapeC), _f32p, _f32p, _f32p]
        L.tko_im2col.argtypes = [C.POINTER(ConvShapeC), _f32p, _f32p]
        L.tko_filter_matrix.argtypes = [C.c_size_t] * 4 + [_f32p, _f32p]
        L.tko_conv2d_winograd.argtypes = [C.POINTER(ConvShapeC), C.c_size_t, _f32p, _f32p, _f32p,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_size_t)]
        L.tko_conv2d_winograd.restype = C.c_int
        L.tko_winograd_plan.argtypes = [C.c_size_t, C.c_size_t, _f32p, _f32p, _f32p]
        L.tko_winograd_plan.restype = C.c_int
        L.tko_max_rel_error.argtypes = [_f32p, _f32p, C.c_size_t, C.c_double]
        L.tko_max_rel_error.restype = C.c_double
        L.tko_max_scaled_error.argtypes = [_f32p, _f32p, C.c_size_t, C.c_double]
        L.tko_max_scaled_error.restype = C.c_double
        _lib = L
    return _lib


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    """The unmodified reference (ref_shim.cpp over /root/reference headers)."""
    global _ref
    if _ref is None:
        if not have_ref():
            raise RuntimeError("oracle/_ref/libtkref.so not built (needs /root/reference)")
        R = C.CDLL(REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_fill_random.argtypes = [_f32p, C.c_size_t, C.c_uint64]
        R.ref_fnv1a.argtypes = [C.c_char_p]
        R.ref_fnv1a.restype = C.c_uint64
        R.ref_gemm_naive.argtypes = [C.c_size_t] * 3 + [C.c_float] * 2 + [C.c_int] * 2 + [_f32p] * 4
        R.ref_gemm_tiled.argtypes = ([C.c_size_t] * 3 + [C.c_float] * 2 + [C.c_int] * 2 +
                                     [_f32p] * 4 + [C.c_char_p, C.c_char_p])
        R.ref_gemm_batched_strided.argtypes = [_f32p, C.c_size_t, _f32p, C.c_size_t, _f32p,
                                               C.c_size_t] + [C.c_size_t] * 4
        R.ref_gemm_batched_strided.restype = C.c_uint64
        R.ref_conv2d.argtypes = [C.POINTER(ConvShapeC), C.c_char_p, _f32p, _f32p, _f32p]
        R.ref_conv2d_winograd.argtypes = [C.POINTER(ConvShapeC), C.c_size_t, _f32p, _f32p, _f32p,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_size_t)]
        R.ref_im2col.argtypes = [C.POINTER(ConvShapeC), _f32p, _f32p]
        R.ref_tune_gemm_stock.argtypes = [C.c_size_t] * 3 + [C.c_int, C.c_int,
                                                             C.POINTER(C.c_int64), C.c_char_p,
                                                             C.c_size_t]
        R.ref_benchmark_conv.argtypes = [C.POINTER(ConvShapeC), C.c_char_p, C.c_int, C.c_int,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        R.ref_time_conv2d.argtypes = [C.POINTER(ConvShapeC), C.c_char_p, _f32p, _f32p, _f32p]
        R.ref_time_conv2d.restype = C.c_int64
        _ref = R
    return _ref


def _check_ref(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {ref().ref_last_error().decode()}")


# ----------------------------------------------------------------------------
# Oracle functions (C restatement)
# ----------------------------------------------------------------------------

def fill_random(count: int, seed: int) -> np.ndarray:
    out = np.empty(count, np.float32)
    lib().tko_fill_random(out, count, seed & 0xFFFFFFFFFFFFFFFF)
    return out


def fnv1a(text: str) -> int:
    return lib().tko_fnv1a(text.encode())


def gemm_naive(m, n, k, alpha, beta, ta, tb, a, b, c) -> np.ndarray:
    out = np.empty(m * n, np.float32)
    cc = c if c is not None else np.zeros(m * n, np.float32)
    lib().tko_gemm_naive(m, n, k, alpha, beta, int(ta), int(tb),
                         np.ascontiguousarray(a, np.float32).ravel(),
                         np.ascontiguousarray(b, np.float32).ravel(),
                         np.ascontiguousarray(cc, np.float32).ravel(), out)
    return out


def gemm_batched_strided(a, b, batch, m, n, k):
    c = np.empty(batch * m * n, np.float32)
    cnt = lib().tko_gemm_batched_strided(np.ascontiguousarray(a, np.float32).ravel(), m * k,
                                         np.ascontiguousarray(b, np.float32).ravel(), k * n,
                                         c, m * n, batch, m, n, k)
    return c, cnt


def conv2d_naive(s: Conv, inp, filt) -> np.ndarray:
    out = np.empty(s.out_shape, np.float32)
    lib().tko_conv2d_naive(C.byref(s.c()), np.ascontiguousarray(inp, np.float32),
                           np.ascontiguousarray(filt, np.float32), out)
    return out


def im2col(s: Conv, inp) -> np.ndarray:
    rows = s.batch * s.out_rows * s.out_cols
    cols = s.window_rows * s.window_cols * s.channels
    out = np.empty(rows * cols, np.float32)
    lib().tko_im2col(C.byref(s.c()), np.ascontiguousarray(inp, np.float32), out)
    return out


def filter_matrix(filt) -> np.ndarray:
    r, s_, c, k = filt.shape
    out = np.empty(r * s_ * c * k, np.float32)
    lib().tko_filter_matrix(r, s_, c, k, np.ascontiguousarray(filt, np.float32), out)
    return out


def conv2d_winograd(s: Conv, m: int, inp, filt):
    out = np.empty(s.out_shape, np.float32)
    mults, tiles = C.c_uint64(0), C.c_size_t(0)
    rc = lib().tko_conv2d_winograd(C.byref(s.c()), m, np.ascontiguousarray(inp, np.float32),
                                   np.ascontiguousarray(filt, np.float32), out,
                                   C.byref(mults), C.byref(tiles))
    if rc != 0:
        raise ValueError(f"winograd oracle rejected the arguments (rc={rc})")
    return out, int(mults.value), int(tiles.value)


def winograd_plan(m: int):
    t = m + 2
    bt = np.empty(t * t, np.float32)
    g = np.empty(t * 3, np.float32)
    at = np.empty(m * t, np.float32)
    if not lib().tko_winograd_plan(m, 3, bt, g, at):
        raise ValueError("no plan")
    return bt.reshape(t, t), g.reshape(t, 3), at.reshape(m, t)


def max_rel_error(values, reference, floor=1e-6) -> float:
    v = np.ascontiguousarray(values, np.float32).ravel()
    r = np.ascontiguousarray(reference, np.float32).ravel()
    assert v.size == r.size
    return lib().tko_max_rel_error(v, r, v.size, floor)


def max_scaled_error(values, reference, floor=1e-6) -> float:
    v = np.ascontiguousarray(values, np.float32).ravel()
    r = np.ascontiguousarray(reference, np.float32).ravel()
    assert v.size == r.size
    return lib().tko_max_scaled_error(v, r, v.size, floor)


# ----------------------------------------------------------------------------
# Reference (ref_shim) functions
# ----------------------------------------------------------------------------

def ref_fill_random(count: int, seed: int) -> np.ndarray:
    out = np.empty(count, np.float32)
    ref().ref_fill_random(out, count, seed & 0xFFFFFFFFFFFFFFFF)
    return out


def ref_gemm_naive(m, n, k, alpha, beta, ta, tb, a, b, c) -> np.ndarray:
    out = np.empty(m * n, np.float32)
    _check_ref(ref().ref_gemm_naive(m, n, k, alpha, beta, int(ta), int(tb), a, b, c, out))
    return out


def ref_gemm_tiled(m, n, k, alpha, beta, ta, tb, a, b, c, cfg: str, dev: str = "") -> np.ndarray:
    out = np.empty(m * n, np.float32)
    _check_ref(ref().ref_gemm_tiled(m, n, k, alpha, beta, int(ta), int(tb), a, b, c, out,
                                    cfg.encode(), dev.encode()))
    return out


def ref_conv2d(s: Conv, params: str, inp, filt) -> np.ndarray:
    out = np.empty(s.out_shape, np.float32)
    _check_ref(ref().ref_conv2d(C.byref(s.c()), params.encode(),
                                np.ascontiguousarray(inp, np.float32),
                                np.ascontiguousarray(filt, np.float32), out))
    return out


def ref_conv2d_winograd(s: Conv, m: int, inp, filt):
    out = np.empty(s.out_shape, np.float32)
    mults, tiles = C.c_uint64(0), C.c_size_t(0)
    _check_ref(ref().ref_conv2d_winograd(C.byref(s.c()), m, np.ascontiguousarray(inp, np.float32),
                                         np.ascontiguousarray(filt, np.float32), out,
                                         C.byref(mults), C.byref(tiles)))
    return out, int(mults.value), int(tiles.value)


def ref_im2col(s: Conv, inp) -> np.ndarray:
    rows = s.batch * s.out_rows * s.out_cols
    cols = s.window_rows * s.window_cols * s.channels
    out = np.empty(rows * cols, np.float32)
    _check_ref(ref().ref_im2col(C.byref(s.c()), np.ascontiguousarray(inp, np.float32), out))
    return out


def ref_gemm_batched_strided(a, b, batch, m, n, k):
    c = np.empty(batch * m * n, np.float32)
    cnt = ref().ref_gemm_batched_strided(a, m * k, b, k * n, c, m * n, batch, m, n, k)
    return c, cnt
