"""Timeline of one tensor-core launch (TK_TC_TRACE): per-CTA globaltimer
stamps of setup, first/last slab arrival, accumulator hand-off, epilogue
drain / store issue, and exit.
    python tools/tc_trace.py gemm M,N,K [tf32|bf16] [tile_n] [split]
    python tools/tc_trace.py conv N,H,C,K,R[,stride] [tf32|bf16]"""
import os
import sys

# The library reads its experiment knobs once, at first use.
os.environ["TK_EXPERIMENTS"] = "1"
os.environ["TK_TC_TRACE"] = "1"

import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05347_b200 as tk  # noqa: E402

kind = sys.argv[1]
dims = [int(v) for v in sys.argv[2].split(",")]
prec = sys.argv[3] if len(sys.argv) > 3 else "tf32"
if kind == "gemm":
    m, n, k = dims
    tn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    sp = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    a = torch.rand(m * k, device="cuda") - 0.5
    b = torch.rand(k * n, device="cuda") - 0.5
    c = torch.empty(m * n, device="cuda")
    shape = tk.GemmShape(m, n, k, 1.0, 0.0, "t", "n")

    def run():
        tk.gemm_dev(a, b, None, c, shape, None,
                    options=tk.exec_options(prec, tile_n=tn, split=sp))
else:
    N, H, C, K, R = dims[:5]
    S = dims[5] if len(dims) > 5 else 1
    shp = tk.ConvShape(N, H, H, C, K, R, R, S, True)
    p = tk.parse_conv_params("im2col")
    x = torch.rand(shp.in_shape, device="cuda")
    f = torch.rand(shp.filt_shape, device="cuda")
    y = torch.empty(shp.out_shape, device="cuda")
    ws = torch.empty(max(tk.conv2d_workspace_size(shp, p, prec), 4) // 4 + 1, device="cuda")
    tk.conv2d_prepare_dev(f, shp, p, ws, precision=prec)

    def run():
        tk.conv2d_run_dev(x, f, y, shp, p, ws, precision=prec)
for _ in range(3):  # every launch prints its timeline (stderr); the last one is warm
    run()
torch.cuda.synchronize()
