"""Golden fixtures for the host-side formats around the hot path, generated
from the UNMODIFIED reference (oracle/_ref/libtkref.so; build container only):

* report.csv / report.json -- render_report (analysis.hpp:157-181) on a
  point set that exercises sorting, dropped failures and every number
  shape of the two formats (%.9g CSV, nlohmann-dump JSON)
* layers.json -- load_layer_rows / serialize_layer_rows (layers.hpp:90-185)
  on well-formed and malformed tables: the serialised table or the exact
  ParseError message

    python tests/golden/make_golden_formats.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as O  # noqa: E402

# (problem, config, oi, gflops, ok)
POINTS = [
    ("gemm_nn_m64_n64_k64", "8x4_8x16_loc", 16.0 / 3.0, 12.3456789, 1),
    ("gemm_nn_m128_n64_k64", "4x4_8x8_loc", 170.666666, 0.000123456, 1),
    ("gemm_nn_m64_n64_k64", "4x4_8x8_loc", 5.0, 98765.4321, 1),
    ("gemm_nn_m64_n64_k64", "broken", 1.0, 2.0, 0),
    ("gemm_tn_m1024_n1024_k1024", "8x8_16x16_loc@tf32", 2048.0 / 12.0, 612345.25, 1),
    ("gemm_nt_m8_n8_k8", "cfg", 0.5, 1.5, 1),
    ("gemm_nn_m1_n1_k1", "tiny", 1.0 / 6.0, 1e-7, 1),
    ("gemm_nn_m2_n2_k2", "huge", 1e20, 1234567890123456.0, 1),
    ("gemm_nn_m3_n3_k3", "exp", 1e16, 123456789012345678.0, 1),
    ("gemm_nn_m4_n4_k4", "small", 0.001, 0.0001, 1),
    ("gemm_nn_m5_n5_k5", "zero", 0.0, 100.0, 1),
    ("gemm_nn_m6_n6_k6", "round", 0.1, 1e15, 1),
]

GOOD_TABLES = [
    "# convnet excerpt\nLayer,Window,Stride,Input,Output\n\n"
    "conv1_1, 3, 1, 224x224x3,  224x224x64\npooled_conv, 3, 2, 112x112x64, 56x56x64\n",
    "Layer,Window,Stride,Input,Output\nconv1,3,1,224x224x3,224x224x64\n"
    "stem,7,2,224x224x3,112x112x64\nreduce,1,1,56x56x256,56x56x64\n",
    "Layer , Window,Stride ,Input,Output,\t\nvalid,3,1,10x10x4,8x8x6\n",
    "Layer,Window,Stride,Input,Output\n",
]
BAD_TABLES = [
    "Layer,Window,Input,Output\n",
    "Layer,Window,Stride,Input,Output\nconv,3,1,224x224,224x224x64\n",
    "Layer,Window,Stride,Input,Output\nconv,3,zero,8x8x1,8x8x1\n",
    "Layer,Window,Stride,Input,Output\nconv,3,1,8x8x1\n",
    "# prologue\nLayer,Window,Stride,Input,Output\nconv,0,1,8x8x1,8x8x1\n",
    "",
    "# only comments\n\n",
    "Layer,Window,Stride,Input,Output\nconv,3,1,16x16x8,13x13x8\n",
    "Layer,Window,Stride,Input,Output\n,3,1,8x8x1,8x8x1\n",
    "Layer,Window,Stride,Input,Output\nconv,3,1,8x8x1x2,8x8x1\n",
    "Layer,Window,Stride,Input,Output\nconv,3,1,8x8x1,8xx1\n",
    "Layer,Window,Stride,Input,Output\nconv,3,1,8x8x1,8x8x1,extra\n",
    "Layer,Window,Stride,Input,Output\nconv,3 1,1,8x8x1,8x8x1\n",
]


def main() -> None:
    O.build()
    R = O.ref()
    R.ref_render_report.restype = C.c_longlong
    R.ref_render_report.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int), C.c_int, C.c_char_p, C.c_size_t]
    R.ref_layer_table.restype = C.c_longlong
    R.ref_layer_table.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t]
    R.ref_last_error.restype = C.c_char_p
    n = len(POINTS)
    probs = (C.c_char_p * n)(*[p[0].encode() for p in POINTS])
    cfgs = (C.c_char_p * n)(*[p[1].encode() for p in POINTS])
    ois = (C.c_double * n)(*[p[2] for p in POINTS])
    gfs = (C.c_double * n)(*[p[3] for p in POINTS])
    oks = (C.c_int * n)(*[p[4] for p in POINTS])
    buf = C.create_string_buffer(1 << 16)
    for fmt, name in ((0, "report.csv"), (1, "report.json")):
        length = R.ref_render_report(n, probs, cfgs, ois, gfs, oks, fmt, buf, len(buf))
        assert 0 <= length < len(buf), R.ref_last_error()
        with open(os.path.join(HERE, name), "wb") as f:
            f.write(buf.value)
    with open(os.path.join(HERE, "report_points.json"), "w") as f:
        json.dump([list(p) for p in POINTS], f, indent=1)
        f.write("\n")
    cases = []
    for text in GOOD_TABLES + BAD_TABLES:
        length = R.ref_layer_table(text.encode(), b"test.csv", buf, len(buf))
        if length < 0:
            cases.append({"text": text, "error": R.ref_last_error().decode()})
        else:
            cases.append({"text": text, "serialized": buf.value.decode()})
    with open(os.path.join(HERE, "layers.json"), "w") as f:
        json.dump(cases, f, indent=1)
        f.write("\n")
    print(f"report.csv/json ({n} points), layers.json ({len(cases)} tables)")


if __name__ == "__main__":
    main()
