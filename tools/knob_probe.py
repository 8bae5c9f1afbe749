"""A/B of an experiment knob on conv layers, timed as bench.py times layers
(graph of 4 x [256 MiB L2 eviction, run phase] minus the eviction alone).
Each knob value runs in its own process (the library reads TK_* once).
    python tools/knob_probe.py TK_EPI_SLOTS 2,4,6,8 vgg_conv1_1,conv1 [tf32]
    python tools/knob_probe.py PROBE_OPTS mode=im2col:split=3,default res4a_branch2b
(PROBE_OPTS values use ':' between options; the worker reads them with ',')."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "--worker":
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_1904_05347_b200 as tk
    from bench import RESNET50, VGG16
    layers, prec = sys.argv[2].split(","), sys.argv[3]
    rows = {n: (3, 1, h, c, k) for n, h, c, k, _ in VGG16}
    rows.update({n: (r, s, h, c, k) for n, r, s, h, c, k, _ in RESNET50})
    flush = torch.empty(64 << 20, device="cuda")
    sink = torch.empty((), device="cuda")
    st = torch.cuda.Stream()

    evict_mode = os.environ.get("PROBE_EVICT", "read")

    def graph_ms(fn, reps=4):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                if evict_mode == "read":
                    torch.sum(flush, dim=0, out=sink)
                elif evict_mode == "write":
                    flush.zero_()
                if fn:
                    fn()
        ts = []
        with torch.cuda.stream(st):
            g.replay()
            for _ in range(5):
                st.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                g.replay()
                b.record(st)
                b.synchronize()
                ts.append(a.elapsed_time(b))
        return float(np.median(ts)) / reps

    base = graph_ms(None)
    out = {}
    for name in layers:
        r, s, h, c, k = rows[name]
        shp = tk.ConvShape(32, h, h, c, k, r, r, s, True)
        im = tk.parse_conv_params("im2col")
        x = torch.rand(shp.in_shape, device="cuda") * 2 - 1
        f = torch.rand(shp.filt_shape, device="cuda") * 2 - 1
        y = torch.empty(shp.out_shape, device="cuda")
        # PROBE_OPTS="mode=im2col,split=3,cluster=1": per-call exec options
        kw = dict(kv.split("=") for kv in os.environ.get("PROBE_OPTS", "").split(",") if kv)
        opts = tk.exec_options(prec, mode=kw.get("mode", "auto"), split=int(kw.get("split", 0)),
                               cluster=int(kw.get("cluster", 0)), stages=int(kw.get("stages", 0)))
        try:
            ws = torch.empty(tk.conv2d_workspace_size(shp, im, options=opts) // 4 + 1, device="cuda")
        except tk.TilekitError:
            out[name] = None
            continue
        tk.conv2d_prepare_dev(f, shp, im, ws, options=opts, stream=st)
        out[name] = round((graph_ms(lambda: tk.conv2d_run_dev(x, f, y, shp, im, ws, options=opts,
                                                              stream=st)) - base) * 1e3, 1)
    print(json.dumps(out))
    sys.exit(0)

knob, values, layers = sys.argv[1], sys.argv[2].split(","), sys.argv[3]
prec = sys.argv[4] if len(sys.argv) > 4 else "tf32"
for v in values:
    env = dict(os.environ, TK_EXPERIMENTS="1",
               **({knob: v.replace(":", ",")} if v != "default" else {}))
    r = subprocess.run([sys.executable, __file__, "--worker", layers, prec], env=env,
                       capture_output=True, text=True)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    print(f"{knob}={v}: {line[-1] if line else r.stderr[-400:]}", flush=True)
