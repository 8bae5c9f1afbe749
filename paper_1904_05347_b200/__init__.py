"""paper_1904_05347_b200 -- B200-native tilekit (tiled GEMM / conv2d).

Python binding of the C ABI in ``include/tk_b200.h`` (libtilekit_b200.so,
built in-tree by ``make -C paper_1904_05347_b200``).  The API mirrors the
reference's C++ entry points (proj/include/tilekit/*.hpp): same names,
argument meaning and error classes, with numpy arrays standing in for
``Matrix`` (column-major, flat ``data`` vector) and ``Tensor4`` (NHWC/HWCK,
C-contiguous).  Device-buffer entry points take torch CUDA tensors.

There is no CPU fallback: importing works anywhere (so shapes, grammars and
budgets can be checked on a CPU box), but every compute call needs the CUDA
library and a B200; if the library is missing the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TK_LIB_PATH") or os.path.join(HERE, "libtilekit_b200.so")  # (TK_LIB_PATH: A/B builds)

# ---------------------------------------------------------------------------
# Errors: one class per reference exception (errors.hpp:9-59)
# ---------------------------------------------------------------------------


class TilekitError(RuntimeError):
    """Base of the tilekit error hierarchy (reference ``tilekit::Error``)."""


class ShapeError(TilekitError):
    pass


class ConfigError(TilekitError):
    pass


class ParseError(TilekitError):
    pass


class CapabilityError(TilekitError):
    pass


class ContractError(TilekitError):
    pass


class IoError(TilekitError):
    pass


class TuningError(TilekitError):
    pass


class DeviceError(TilekitError):
    """The B200 failed or is absent (no reference counterpart)."""


_ERRORS = {1: ShapeError, 2: ConfigError, 3: ParseError, 4: CapabilityError,
           5: ContractError, 6: IoError, 7: TuningError, 8: DeviceError}

PREC_FP32_EXACT, PREC_TF32, PREC_BF16, PREC_3XTF32 = 0, 1, 2, 3
PRECISIONS = {"fp32": PREC_FP32_EXACT, "tf32": PREC_TF32, "bf16": PREC_BF16, "3xtf32": PREC_3XTF32}

# ---------------------------------------------------------------------------
# C structs (tk_b200.h)
# ---------------------------------------------------------------------------


class GemmShapeC(C.Structure):
    _fields_ = [("m", C.c_size_t), ("n", C.c_size_t), ("k", C.c_size_t),
                ("alpha", C.c_float), ("beta", C.c_float), ("op_a", C.c_int), ("op_b", C.c_int)]


class GemmConfigC(C.Structure):
    _fields_ = [("reg_rows", C.c_size_t), ("reg_cols", C.c_size_t), ("wg_rows", C.c_size_t),
                ("wg_cols", C.c_size_t), ("use_local_memory", C.c_int),
                ("double_buffer", C.c_int), ("k_step", C.c_size_t)]


class DeviceSpecC(C.Structure):
    _fields_ = [("name", C.c_char_p), ("cache_line_bytes", C.c_size_t),
                ("local_memory_bytes", C.c_size_t), ("compute_units", C.c_size_t),
                ("register_budget", C.c_size_t), ("max_workgroup_size", C.c_size_t)]


class ConvShapeC(C.Structure):
    _fields_ = [("batch", C.c_size_t), ("in_rows", C.c_size_t), ("in_cols", C.c_size_t),
                ("channels", C.c_size_t), ("features", C.c_size_t),
                ("window_rows", C.c_size_t), ("window_cols", C.c_size_t),
                ("stride", C.c_size_t), ("padding", C.c_int)]


class ConvParamsC(C.Structure):
    _fields_ = [("algo", C.c_int), ("tile_rows", C.c_size_t), ("tile_cols", C.c_size_t),
                ("channel_vector", C.c_size_t), ("feature_vector", C.c_size_t)]


class ExecOptionsC(C.Structure):
    _fields_ = [("precision", C.c_int), ("tc_tile_n", C.c_int), ("tc_stages", C.c_int),
                ("tc_cluster", C.c_int), ("tc_mode", C.c_int), ("tc_split", C.c_int),
                ("io", C.c_int), ("reserved", C.c_int * 1)]


# tk_exec_options.io (tk_io_flags): bf16 activations in HBM
IO_FLAGS = {"fp32": 0, "in_bf16": 1, "out_bf16": 2, "bf16": 3}


class ConvPlanInfoC(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "kernel", "precision", "requested_precision", "cta_group", "tile_m", "tile_n", "splits",
        "tail_pieces", "imgs", "flat", "box_w", "box_h", "halo_resident", "winograd_m", "tuned")] + \
        [("reserved", C.c_int * 3)]


class GemmPlanC(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "kernel", "precision", "requested_precision", "cta_group", "tile_m", "tile_n", "splits",
        "tail_pieces", "a_in_place", "b_in_place", "k_depth", "tuned")] + \
        [("reserved", C.c_int * 4)]


KERNELS = {0: "exact_simt", 1: "tc_halo", 2: "tc_pixn", 3: "tc_pixm", 4: "tc_gather",
           5: "tc_pointwise", 6: "tc_im2col", 7: "winograd", 8: "tc_halo_narrow", 9: "tc_plain"}
PRECISION_NAMES = {v: k for k, v in PRECISIONS.items()}


# Every symbol the header declares (checked by the CPU tests).
EXPORTS = [
    "tk_last_error", "tk_abi_version", "tk_device_count", "tk_b200_device_spec",
    "tk_launch_count", "tk_synchronize", "tk_validate_gemm_config", "tk_local_mem_elems",
    "tk_gemm_tiled", "tk_gemm_naive", "tk_gemm_batched_strided", "tk_gemm_dev",
    "tk_gemm_batched_strided_dev", "tk_conv2d", "tk_conv2d_naive", "tk_conv2d_tiled",
    "tk_conv2d_im2col", "tk_conv2d_winograd", "tk_im2col", "tk_filter_matrix",
    "tk_conv2d_dev", "tk_conv2d_workspace_size", "tk_conv2d_ex", "tk_im2col_dev",
    "tk_bench_gemm", "tk_bench_conv2d", "tk_gemm_ex", "tk_conv2d_prepare_dev",
    "tk_conv2d_run_dev", "tk_conv2d_plan_info", "tk_tuning_db_load", "tk_tuning_db_clear",
    "tk_tuning_db_size", "tk_gemm_plan_info",
]

_lib: Optional[C.CDLL] = None

_f32p = C.POINTER(C.c_float)
_vp = C.c_void_p


def lib() -> C.CDLL:
    """Load libtilekit_b200.so; raises (no fallback) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"{LIB_PATH} is not built: run `make -C {HERE}` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.tk_last_error.restype = C.c_char_p
    L.tk_launch_count.restype = C.c_uint64
    sig = {
        "tk_b200_device_spec": [C.POINTER(DeviceSpecC)],
        "tk_validate_gemm_config": [C.POINTER(GemmConfigC), C.POINTER(DeviceSpecC),
                                    C.POINTER(C.c_int), C.c_char_p, C.c_size_t],
        "tk_local_mem_elems": [C.POINTER(GemmConfigC), C.POINTER(DeviceSpecC),
                               C.POINTER(C.c_size_t)],
        "tk_gemm_tiled": [C.POINTER(GemmShapeC), C.POINTER(GemmConfigC), C.POINTER(DeviceSpecC),
                          _vp, _vp, _vp, _vp],
        "tk_gemm_naive": [C.POINTER(GemmShapeC), _vp, _vp, _vp, _vp],
        "tk_gemm_batched_strided": [_vp, C.c_size_t, _vp, C.c_size_t, _vp, C.c_size_t,
                                    C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                    C.POINTER(C.c_uint64)],
        "tk_gemm_dev": [C.POINTER(GemmShapeC), C.POINTER(GemmConfigC),
                        C.POINTER(ExecOptionsC), _vp, _vp, _vp, _vp, _vp],
        "tk_gemm_batched_strided_dev": [_vp, C.c_size_t, _vp, C.c_size_t, _vp, C.c_size_t,
                                        C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                        C.POINTER(ExecOptionsC), _vp],
        "tk_conv2d": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC), _vp, _vp, _vp],
        "tk_conv2d_ex": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC),
                         C.POINTER(ExecOptionsC), _vp, _vp, _vp],
        "tk_conv2d_naive": [C.POINTER(ConvShapeC), _vp, _vp, _vp],
        "tk_conv2d_tiled": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC), _vp, _vp, _vp],
        "tk_conv2d_im2col": [C.POINTER(ConvShapeC), C.POINTER(GemmConfigC),
                             C.POINTER(DeviceSpecC), _vp, _vp, _vp],
        "tk_conv2d_winograd": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC), _vp, _vp, _vp,
                               C.POINTER(C.c_uint64), C.POINTER(C.c_size_t)],
        "tk_im2col": [C.POINTER(ConvShapeC), _vp, _vp],
        "tk_im2col_dev": [C.POINTER(ConvShapeC), _vp, _vp, _vp],
        "tk_filter_matrix": [C.c_size_t] * 4 + [_vp, _vp],
        "tk_conv2d_dev": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC),
                          C.POINTER(ExecOptionsC), _vp, _vp, _vp, _vp, C.c_size_t, _vp],
        "tk_conv2d_workspace_size": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC),
                                     C.POINTER(ExecOptionsC), C.POINTER(C.c_size_t)],
        "tk_conv2d_prepare_dev": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC),
                                  C.POINTER(ExecOptionsC), _vp, _vp, C.c_size_t, _vp],
        "tk_conv2d_run_dev": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC),
                              C.POINTER(ExecOptionsC), _vp, _vp, _vp, _vp, C.c_size_t, _vp],
        "tk_conv2d_plan_info": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC),
                                C.POINTER(ExecOptionsC), C.POINTER(ConvPlanInfoC)],
        "tk_tuning_db_load": [C.c_char_p, C.c_char_p, C.POINTER(C.c_size_t)],
        "tk_gemm_plan_info": [C.POINTER(GemmShapeC), C.POINTER(GemmConfigC),
                              C.POINTER(ExecOptionsC), C.POINTER(GemmPlanC)],
        "tk_tuning_db_clear": [],
        "tk_tuning_db_size": [C.POINTER(C.c_size_t)],
        "tk_gemm_ex": [C.POINTER(GemmShapeC), C.POINTER(ExecOptionsC), _vp, _vp, _vp, _vp],
        "tk_bench_gemm": [C.POINTER(GemmShapeC), C.POINTER(GemmConfigC), C.POINTER(ExecOptionsC),
                          _vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(C.c_int64)],
        "tk_bench_conv2d": [C.POINTER(ConvShapeC), C.POINTER(ConvParamsC),
                            C.POINTER(ExecOptionsC), _vp, _vp, C.c_int, C.c_int,
                            C.POINTER(C.c_int64)],
    }
    for name, args in sig.items():
        getattr(L, name).argtypes = args
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().tk_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, DeviceError)(msg)


def device_count() -> int:
    return lib().tk_device_count()


def launch_count() -> int:
    return int(lib().tk_launch_count())


# ---------------------------------------------------------------------------
# Parameter structs + grammars (reference config.hpp:19-290)
# ---------------------------------------------------------------------------


@dataclass
class GemmShape:
    m: int
    n: int
    k: int
    alpha: float = 1.0
    beta: float = 0.0
    op_a: str = "n"  # 'n' Identity, 't' Transpose
    op_b: str = "n"

    def c(self) -> GemmShapeC:
        return GemmShapeC(self.m, self.n, self.k, self.alpha, self.beta,
                          int(self.op_a == "t"), int(self.op_b == "t"))

    def flops(self) -> int:
        return 2 * self.m * self.n * self.k

    def key(self) -> str:
        return f"gemm_{self.op_a}{self.op_b}_m{self.m}_n{self.n}_k{self.k}"


@dataclass
class GemmConfig:
    reg_rows: int = 4
    reg_cols: int = 4
    wg_rows: int = 8
    wg_cols: int = 8
    use_local_memory: bool = False
    double_buffer: bool = False
    k_step: int = 1

    def c(self) -> GemmConfigC:
        return GemmConfigC(self.reg_rows, self.reg_cols, self.wg_rows, self.wg_cols,
                           int(self.use_local_memory), int(self.double_buffer), self.k_step)

    def name(self) -> str:
        s = (f"{self.reg_rows}x{self.reg_cols}_{self.wg_rows}x{self.wg_cols}_"
             f"{'loc' if self.use_local_memory else 'noloc'}")
        return s + ("_db" if self.double_buffer else "")


def parse_gemm_config(text: str) -> GemmConfig:
    """Grammar ``{h}x{w}_{r}x{c}_{loc|noloc}[_db]`` (config.hpp:96-131)."""
    import re
    m = re.fullmatch(r"([1-9]\d*)x([1-9]\d*)_([1-9]\d*)x([1-9]\d*)_(loc|noloc)(_db)?", text)
    if not m or (m.group(6) and m.group(5) != "loc"):
        raise ParseError(f'config name "{text}": malformed')
    return GemmConfig(int(m.group(1)), int(m.group(2)), int(m.group(3)), int(m.group(4)),
                      m.group(5) == "loc", bool(m.group(6)))


@dataclass
class DeviceSpec:
    name: str
    cache_line_bytes: int = 64
    local_memory_bytes: int = 0
    compute_units: int = 1
    register_budget: int = 256
    max_workgroup_size: int = 256

    def c(self) -> DeviceSpecC:
        self._name = self.name.encode()
        return DeviceSpecC(self._name, self.cache_line_bytes, self.local_memory_bytes,
                           self.compute_units, self.register_budget, self.max_workgroup_size)


BUILTIN_DEVICES = [
    DeviceSpec("Intel Core i7-6700K CPU", 64, 0, 8),
    DeviceSpec("Intel Core i7-6700K GPU", 64, 64 * 1024, 24),
    DeviceSpec("ARM Mali G71 GPU", 64, 0, 8),
    DeviceSpec("Renesas V3M", 128, 447 * 1024, 2),
    DeviceSpec("Renesas V3H", 128, 409 * 1024, 5),
    DeviceSpec("AMD R9 Nano", 128, 32 * 1024, 64),
]


def find_device(name: str) -> DeviceSpec:
    canon = lambda s: "".join(ch.lower() for ch in s if ch not in " -_")  # noqa: E731
    want = canon(name)
    hits = [d for d in BUILTIN_DEVICES if canon(d.name) == want]
    if hits:
        return hits[0]
    hits = [d for d in BUILTIN_DEVICES if want and want in canon(d.name)]
    if len(hits) != 1:
        raise ParseError(f'{"ambiguous" if hits else "unknown"} device "{name}"')
    return hits[0]


def b200_device() -> DeviceSpec:
    s = DeviceSpecC()
    _check(lib().tk_b200_device_spec(C.byref(s)))
    return DeviceSpec(s.name.decode(), s.cache_line_bytes, s.local_memory_bytes,
                      s.compute_units, s.register_budget, s.max_workgroup_size)


def validate_config(cfg: GemmConfig, dev: DeviceSpec):
    """(ok, summary) of validate_config (gemm.hpp:103-146)."""
    ok = C.c_int(0)
    buf = C.create_string_buffer(4096)
    _check(lib().tk_validate_gemm_config(C.byref(cfg.c()), C.byref(dev.c()), C.byref(ok), buf,
                                         4096))
    return bool(ok.value), buf.value.decode()


@dataclass
class ConvShape:
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
        return ConvShapeC(self.batch, self.in_rows, self.in_cols, self.channels, self.features,
                          self.window_rows, self.window_cols, self.stride, int(self.same))

    def _out(self, n, w):
        if not self.same:
            return 0 if n < w else (n - w) // self.stride + 1
        return (n + self.stride - 1) // self.stride

    @property
    def out_rows(self):
        return self._out(self.in_rows, self.window_rows)

    @property
    def out_cols(self):
        return self._out(self.in_cols, self.window_cols)

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
        """conv_flops (conv.hpp:19-23)."""
        return (2 * self.batch * self.out_rows * self.out_cols * self.features *
                self.window_rows * self.window_cols * self.channels)

    def key(self) -> str:
        return (f"conv_n{self.batch}_{self.in_rows}x{self.in_cols}x{self.channels}"
                f"_k{self.features}_f{self.window_rows}x{self.window_cols}"
                f"_s{self.stride}_{'same' if self.same else 'valid'}")


ALGOS = {"naive": 0, "tiled": 1, "im2col": 2, "winograd": 3}


@dataclass
class ConvAlgoParams:
    algo: str = "naive"
    tile_rows: int = 1
    tile_cols: int = 1
    channel_vector: int = 1
    feature_vector: int = 1

    def c(self) -> ConvParamsC:
        return ConvParamsC(ALGOS[self.algo], self.tile_rows, self.tile_cols,
                           self.channel_vector, self.feature_vector)

    def name(self) -> str:
        if self.algo in ("naive", "im2col"):
            return self.algo
        if self.algo == "winograd":
            return f"winograd_t{self.tile_rows}x{self.tile_cols}"
        return (f"tiled_t{self.tile_rows}x{self.tile_cols}_v{self.channel_vector}"
                f"x{self.feature_vector}")


def parse_conv_params(text: str) -> ConvAlgoParams:
    """Grammar of parse_conv_params (config.hpp:247-290)."""
    import re
    if text in ("naive", "im2col"):
        return ConvAlgoParams(text)
    m = re.fullmatch(r"winograd_t([1-9]\d*)x([1-9]\d*)", text)
    if m:
        return ConvAlgoParams("winograd", int(m.group(1)), int(m.group(2)))
    m = re.fullmatch(r"tiled_t([1-9]\d*)x([1-9]\d*)_v([1-9]\d*)x([1-9]\d*)", text)
    if m:
        cv, fv = int(m.group(3)), int(m.group(4))
        if cv not in (1, 2, 4, 8) or fv not in (1, 2, 4, 8):
            raise ParseError(f'conv params "{text}": vector widths must be one of 1, 2, 4, 8')
        return ConvAlgoParams("tiled", int(m.group(1)), int(m.group(2)), cv, fv)
    raise ParseError(f'conv params "{text}": unrecognized name')


TC_MODES = {"auto": 0, "halo": 1, "pixn": 2, "pixm": 3, "gather": 4, "pointwise": 5, "im2col": 6}


def exec_options(precision="fp32", tile_n=0, stages=0, cluster=0, mode="auto",
                 split=0, io="fp32") -> ExecOptionsC:
    """io: "fp32" (the reference's fp32 NHWC in/out), or -- with precision
    "bf16" and the im2col algorithm -- "in_bf16" / "out_bf16" / "bf16":
    the input and/or output activations are bf16 tensors in HBM (a BF16
    network's layer-to-layer format; no conversion pass)."""
    p = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
    m = TC_MODES[mode] if isinstance(mode, str) else int(mode)
    f = IO_FLAGS[io] if isinstance(io, str) else int(io)
    return ExecOptionsC(p, tile_n, stages, cluster, m, split, f)


# ---------------------------------------------------------------------------
# Host-buffer API (numpy in, numpy out): the reference function surface
# ---------------------------------------------------------------------------


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# Operand checks before any pointer crosses the C ABI (the reference raises
# ShapeError from check_gemm_operands / check_conv_operands, gemm.hpp:165-186,
# conv.hpp:30-66): an undersized buffer must never be read past its end.
def _need_size(arr, count: int, what: str) -> None:
    n = int(arr.size) if isinstance(arr, np.ndarray) else int(arr.numel())
    if n != count:
        raise ShapeError(f"{what} has {n} elements, expected {count}")


def _gemm_sizes(shape: "GemmShape"):
    return shape.m * shape.k, shape.k * shape.n, shape.m * shape.n


def _need_shape(arr, want, what: str) -> None:
    got = tuple(arr.shape)
    if got != tuple(want):
        if int(np.prod(got)) == int(np.prod(want)) and len(got) == 1:
            return  # flat buffer of the right size
        raise ShapeError(f"conv2d: {what} is {'x'.join(map(str, got))}, expected "
                         f"{'x'.join(map(str, want))}")


def _need_dev(t, what: str, count: Optional[int] = None, dtype_f32: bool = True,
              bf16: bool = False) -> None:
    """Device operand: a contiguous CUDA tensor (float32 -- bfloat16 for bf16
    activations -- unless a workspace) holding exactly `count` elements (at
    least, for workspaces: count=None)."""
    if t is None:
        return
    if not getattr(t, "is_cuda", False):
        raise ContractError(f"{what} must be a CUDA tensor")
    if dtype_f32:
        import torch
        want = torch.bfloat16 if bf16 else torch.float32
        if t.dtype != want:
            raise ContractError(f"{what} must be {str(want).split('.')[-1]}, got {t.dtype}")
    if not t.is_contiguous():
        raise ContractError(f"{what} must be contiguous")
    if count is not None and t.numel() != count:
        raise ShapeError(f"{what} has {t.numel()} elements, expected {count}")


def gemm_tiled(a, b, c, shape: GemmShape, cfg: GemmConfig, dev: DeviceSpec) -> np.ndarray:
    """gemm_tiled (gemm.hpp:308): flat column-major operands, returns m*n."""
    a, b = _f32(a).ravel(), _f32(b).ravel()
    c = _f32(c).ravel() if c is not None else np.zeros(shape.m * shape.n, np.float32)
    na, nb, nc = _gemm_sizes(shape)
    _need_size(a, na, "gemm: operand A")
    _need_size(b, nb, "gemm: operand B")
    _need_size(c, nc, "gemm: operand C")
    out = np.empty(shape.m * shape.n, np.float32)
    _check(lib().tk_gemm_tiled(C.byref(shape.c()), C.byref(cfg.c()), C.byref(dev.c()),
                               _ptr(a), _ptr(b), _ptr(c), _ptr(out)))
    return out


def gemm_naive(a, b, c, shape: GemmShape) -> np.ndarray:
    a, b = _f32(a).ravel(), _f32(b).ravel()
    c = _f32(c).ravel() if c is not None else np.zeros(shape.m * shape.n, np.float32)
    na, nb, nc = _gemm_sizes(shape)
    _need_size(a, na, "gemm: operand A")
    _need_size(b, nb, "gemm: operand B")
    _need_size(c, nc, "gemm: operand C")
    out = np.empty(shape.m * shape.n, np.float32)
    _check(lib().tk_gemm_naive(C.byref(shape.c()), _ptr(a), _ptr(b), _ptr(c), _ptr(out)))
    return out


def gemm_batched_strided(a, b, batch, m, n, k):
    """C_g = A_g B_g over packed column-major members; returns (c, multiplies)."""
    a, b = _f32(a).ravel(), _f32(b).ravel()
    _need_size(a, batch * m * k, "gemm_batched_strided: operand A")
    _need_size(b, batch * k * n, "gemm_batched_strided: operand B")
    c = np.zeros(batch * m * n, np.float32)
    cnt = C.c_uint64(0)
    _check(lib().tk_gemm_batched_strided(_ptr(a), m * k, _ptr(b), k * n, _ptr(c), m * n,
                                         batch, m, n, k, C.byref(cnt)))
    return c, int(cnt.value)


def gemm_batched_strided_dev(a, b, c, batch, m, n, k, precision="fp32", stream=None,
                             options=None) -> None:
    """gemm_batched_strided (gemm.hpp:451-479) on device buffers: C_g = A_g B_g
    over packed column-major members (strides m*k, k*n, m*n).  fp32: the
    bit-exact SIMT path; tf32 / bf16 / 3xtf32: one batched tensor-core GEMM
    (3xTF32 member by member)."""
    opts = options if options is not None else exec_options(precision)
    _need_dev(a, "gemm_batched_strided: operand A", batch * m * k)
    _need_dev(b, "gemm_batched_strided: operand B", batch * k * n)
    _need_dev(c, "gemm_batched_strided: output", batch * m * n)
    _check(lib().tk_gemm_batched_strided_dev(_dptr(a), m * k, _dptr(b), k * n, _dptr(c), m * n,
                                             batch, m, n, k, C.byref(opts), _stream(stream)))


def conv2d(inp, filt, shape: ConvShape, params: ConvAlgoParams, precision="fp32") -> np.ndarray:
    """conv2d selector (winograd.hpp:304); precision != fp32 uses tensor cores."""
    inp, filt = _f32(inp), _f32(filt)
    _need_shape(inp, shape.in_shape, "input")
    _need_shape(filt, shape.filt_shape, "filter")
    out = np.empty(shape.out_shape, np.float32)
    if precision == "fp32":
        rc = lib().tk_conv2d(C.byref(shape.c()), C.byref(params.c()), _ptr(inp), _ptr(filt),
                             _ptr(out))
    else:
        rc = lib().tk_conv2d_ex(C.byref(shape.c()), C.byref(params.c()),
                                C.byref(exec_options(precision)), _ptr(inp), _ptr(filt),
                                _ptr(out))
    _check(rc)
    return out


def conv2d_im2col(inp, filt, shape: ConvShape, cfg: GemmConfig, dev: DeviceSpec) -> np.ndarray:
    inp, filt = _f32(inp), _f32(filt)
    _need_shape(inp, shape.in_shape, "input")
    _need_shape(filt, shape.filt_shape, "filter")
    out = np.empty(shape.out_shape, np.float32)
    _check(lib().tk_conv2d_im2col(C.byref(shape.c()), C.byref(cfg.c()), C.byref(dev.c()),
                                  _ptr(inp), _ptr(filt), _ptr(out)))
    return out


def conv2d_winograd(inp, filt, shape: ConvShape, params: ConvAlgoParams):
    inp, filt = _f32(inp), _f32(filt)
    _need_shape(inp, shape.in_shape, "input")
    _need_shape(filt, shape.filt_shape, "filter")
    out = np.empty(shape.out_shape, np.float32)
    mults, tiles = C.c_uint64(0), C.c_size_t(0)
    _check(lib().tk_conv2d_winograd(C.byref(shape.c()), C.byref(params.c()), _ptr(inp),
                                    _ptr(filt), _ptr(out), C.byref(mults), C.byref(tiles)))
    return out, int(mults.value), int(tiles.value)


def im2col(inp, shape: ConvShape) -> np.ndarray:
    inp = _f32(inp)
    _need_shape(inp, shape.in_shape, "input")
    rows = shape.batch * shape.out_rows * shape.out_cols
    cols = shape.window_rows * shape.window_cols * shape.channels
    out = np.empty(rows * cols, np.float32)
    _check(lib().tk_im2col(C.byref(shape.c()), _ptr(inp), _ptr(out)))
    return out


def filter_matrix(filt) -> np.ndarray:
    filt = _f32(filt)
    r, s, c, k = filt.shape
    out = np.empty(r * s * c * k, np.float32)
    _check(lib().tk_filter_matrix(r, s, c, k, _ptr(filt), _ptr(out)))
    return out


# ---------------------------------------------------------------------------
# Device-buffer API (torch CUDA tensors; caller owns memory and stream)
# ---------------------------------------------------------------------------


def _dptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream(stream) -> C.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _need_conv_dev(shape: ConvShape, inp, filt, out, workspace, io: int = 0) -> None:
    _need_dev(inp, "conv2d: input", int(np.prod(shape.in_shape)), bf16=bool(io & 1))
    _need_dev(filt, "conv2d: filter", int(np.prod(shape.filt_shape)))
    _need_dev(out, "conv2d: output", int(np.prod(shape.out_shape)), bf16=bool(io & 2))
    _need_dev(workspace, "conv2d: workspace", None, dtype_f32=False)


def conv2d_dev(inp, filt, out, shape: ConvShape, params: ConvAlgoParams, precision="fp32",
               workspace=None, stream=None, tile_n=0, options=None) -> None:
    """options: an exec_options(...) record (tensor-core knobs); overrides
    precision / tile_n when given."""
    opts = options if options is not None else exec_options(precision, tile_n)
    _need_conv_dev(shape, inp, filt, out, workspace, opts.io)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().tk_conv2d_dev(C.byref(shape.c()), C.byref(params.c()),
                               C.byref(opts), _dptr(inp), _dptr(filt),
                               _dptr(out), _dptr(workspace), ws_bytes, _stream(stream)))


def conv2d_prepare_dev(filt, shape: ConvShape, params: ConvAlgoParams, workspace,
                       precision="fp32", stream=None, options=None) -> None:
    """Filter-side phase of conv2d_dev (may run on its own stream)."""
    _need_conv_dev(shape, None, filt, None, workspace)
    ws_bytes = workspace.numel() * workspace.element_size()
    opts = options if options is not None else exec_options(precision)
    _check(lib().tk_conv2d_prepare_dev(C.byref(shape.c()), C.byref(params.c()),
                                       C.byref(opts), _dptr(filt),
                                       _dptr(workspace), ws_bytes, _stream(stream)))


def conv2d_run_dev(inp, filt, out, shape: ConvShape, params: ConvAlgoParams, workspace,
                   precision="fp32", stream=None, options=None) -> None:
    """Input-side phase of conv2d_dev; ordered after conv2d_prepare_dev."""
    opts = options if options is not None else exec_options(precision)
    _need_conv_dev(shape, inp, filt, out, workspace, opts.io)
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().tk_conv2d_run_dev(C.byref(shape.c()), C.byref(params.c()),
                                   C.byref(opts), _dptr(inp), _dptr(filt),
                                   _dptr(out), _dptr(workspace), ws_bytes, _stream(stream)))


def conv2d_workspace_size(shape: ConvShape, params: ConvAlgoParams, precision="fp32",
                          options=None) -> int:
    n = C.c_size_t(0)
    opts = options if options is not None else exec_options(precision)
    _check(lib().tk_conv2d_workspace_size(C.byref(shape.c()), C.byref(params.c()),
                                          C.byref(opts), C.byref(n)))
    return int(n.value)


def conv2d_plan_info(shape: ConvShape, params: ConvAlgoParams, precision="fp32",
                     options=None) -> dict:
    """The plan conv2d_dev runs for this call (tk_conv2d_plan_info): kernel
    family, EFFECTIVE precision (a BF16 request on a path without BF16
    operands reports tf32), tile and work split.  Host-side only."""
    info = ConvPlanInfoC()
    opts = options if options is not None else exec_options(precision)
    _check(lib().tk_conv2d_plan_info(C.byref(shape.c()), C.byref(params.c()), C.byref(opts),
                                     C.byref(info)))
    d = {f: getattr(info, f) for f, _ in ConvPlanInfoC._fields_ if f != "reserved"}
    d["kernel"] = KERNELS[d["kernel"]]
    d["precision"] = PRECISION_NAMES[d["precision"]]
    d["requested_precision"] = PRECISION_NAMES[d["requested_precision"]]
    return d


def gemm_plan_info(shape: GemmShape, cfg: Optional[GemmConfig] = None, precision="fp32",
                   options=None) -> dict:
    """The plan gemm_dev runs for this call (tk_gemm_plan_info): kernel
    family, effective precision, CTA group, tile, split-K / stream-K tail,
    which operands are read in place, whether the tuning DB chose the knobs.
    Host-side only (operands assumed 16-byte aligned)."""
    info = GemmPlanC()
    opts = options if options is not None else exec_options(precision)
    _check(lib().tk_gemm_plan_info(C.byref(shape.c()), C.byref(cfg.c()) if cfg is not None else None,
                                   C.byref(opts), C.byref(info)))
    d = {f: getattr(info, f) for f, _ in GemmPlanC._fields_ if f != "reserved"}
    d["kernel"] = KERNELS[d["kernel"]]
    d["precision"] = PRECISION_NAMES[d["precision"]]
    d["requested_precision"] = PRECISION_NAMES[d["requested_precision"]]
    return d


def tuning_db_load(path: str, device: Optional[str] = None) -> int:
    """Load the tuner's NDJSON DB into the library (lookup_best on the launch
    path): calls with automatic tensor-core knobs then run the fastest
    recorded knobs for their problem.  Returns the records kept."""
    n = C.c_size_t(0)
    _check(lib().tk_tuning_db_load(path.encode(), device.encode() if device else None, C.byref(n)))
    return int(n.value)


def tuning_db_clear() -> None:
    _check(lib().tk_tuning_db_clear())


def tuning_db_size() -> int:
    n = C.c_size_t(0)
    _check(lib().tk_tuning_db_size(C.byref(n)))
    return int(n.value)


def gemm_dev(a, b, c, out, shape: GemmShape, cfg: Optional[GemmConfig] = None,
             precision="fp32", stream=None, tile_n=0, options=None) -> None:
    """options: an exec_options(...) record (tensor-core knobs); overrides
    precision / tile_n when given.  exec_options("bf16", io="in_bf16"): A and
    B are bfloat16 tensors (bf16 operands in HBM); C and out stay float32."""
    opts = options if options is not None else exec_options(precision, tile_n)
    na, nb, nc = _gemm_sizes(shape)
    _need_dev(a, "gemm: operand A", na, bf16=bool(opts.io & 1))
    _need_dev(b, "gemm: operand B", nb, bf16=bool(opts.io & 1))
    if shape.beta != 0.0:
        if c is None:
            raise ContractError("gemm: beta != 0 needs operand C")
        _need_dev(c, "gemm: operand C", nc)
    _need_dev(out, "gemm: output", nc)
    cfg_c = C.byref(cfg.c()) if cfg is not None else None
    _check(lib().tk_gemm_dev(C.byref(shape.c()), cfg_c, C.byref(opts),
                             _dptr(a), _dptr(b), _dptr(c), _dptr(out), _stream(stream)))


def im2col_dev(inp, out, shape: ConvShape, stream=None) -> None:
    _need_dev(inp, "conv2d: input", int(np.prod(shape.in_shape)))
    _need_dev(out, "im2col: patches", shape.batch * shape.out_rows * shape.out_cols *
              shape.window_rows * shape.window_cols * shape.channels)
    _check(lib().tk_im2col_dev(C.byref(shape.c()), _dptr(inp), _dptr(out), _stream(stream)))
