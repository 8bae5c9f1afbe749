"""Per-layer ncu counters of the bench's conv layers (batch 32, the bench's
plans): every distinct VGG16 / ResNet-50 shape runs its run phase once
between marker fills, so a launch list of this script attributes each
kernel to its layer.

    # GPU box:
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,\
dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv \
        --log-file launches.csv python tools/layer_ncu.py run tf32
    # here:
    python tools/layer_ncu.py summarise launches.csv tf32 > profiles/rNN_layer_ncu_tf32.txt
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def shapes():
    from bench import RESNET50, VGG16
    out = [(n, 3, 1, h, c, k) for n, h, c, k, _ in VGG16]
    out += [(n, r, s, h, c, k) for n, r, s, h, c, k, _ in RESNET50]
    return out


def run(prec):
    import torch
    import paper_1904_05347_b200 as tk
    db = os.path.join(ROOT, "profiles", "r02_tune_ncu.ndjson")
    if os.path.exists(db):
        tk.tuning_db_load(db)
    marker = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.Stream()
    im = tk.parse_conv_params("im2col")
    with torch.cuda.stream(st):
        for i, (name, r, s, h, c, k) in enumerate(shapes()):
            shp = tk.ConvShape(32, h, h, c, k, r, r, s, True)
            x = torch.rand(shp.in_shape, device="cuda") * 2 - 1
            f = torch.rand(shp.filt_shape, device="cuda") * 2 - 1
            y = torch.empty(shp.out_shape, device="cuda")
            ws = torch.empty(tk.conv2d_workspace_size(shp, im, prec) // 4 + 1, device="cuda")
            tk.conv2d_prepare_dev(f, shp, im, ws, precision=prec, stream=st)
            tk.conv2d_run_dev(x, f, y, shp, im, ws, precision=prec, stream=st)  # warm
            marker.fill_(i + 1)  # FillFunctor<long>: layer delimiter
            tk.conv2d_run_dev(x, f, y, shp, im, ws, precision=prec, stream=st)
            marker.fill_(-1)
            st.synchronize()
            del x, f, y, ws


def summarise(path, prec):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im_, iv, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                        hdr.index("Metric Value"), hdr.index("ID"))
    launches = {}
    for r in rows[1:]:
        d = launches.setdefault(int(r[iid]), {"kernel": r[ik]})
        d[r[im_]] = float(r[iv].replace(",", ""))
    seq = [launches[i] for i in sorted(launches)]
    first = next(i for i, d in enumerate(seq) if "FillFunctor<long" in d["kernel"])
    seq = seq[first + 1:]  # (the marker's own zero fill)
    names = [s[0] for s in shapes()]
    layer, idx, out = None, 0, {}
    for d in seq:
        if "FillFunctor<long" in d["kernel"]:
            if layer is None:
                layer = names[idx]
                idx += 1
                out[layer] = []
            else:
                layer = None
            continue
        if layer is not None:
            out[layer].append(d)
    print(f"# per-layer ncu counters, {prec}, batch 32 (tools/layer_ncu.py; cold L2, serialised)")
    print(f"{'layer':16s} {'us':>7s} {'DRAM MB':>8s} {'dram%':>6s} {'tensor%':>7s}  kernels")
    total = {}
    for name, ks in out.items():
        t = sum(k.get("gpu__time_duration.sum", 0) for k in ks) / 1e3
        mb = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks) / 1e6
        main = max(ks, key=lambda k: k.get("gpu__time_duration.sum", 0)) if ks else {}
        dr = main.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0)
        tp = main.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
        kn = ", ".join(f"{k['kernel'].split('(')[0].replace('void ', '').replace('tkb::<unnamed>::', '')}"
                       f" {k.get('gpu__time_duration.sum', 0) / 1e3:.1f}" for k in ks)
        print(f"{name:16s} {t:7.1f} {mb:8.1f} {dr:6.1f} {tp:7.1f}  {kn}")
        total[name] = {"us": round(t, 2), "dram_mb": round(mb, 2), "main_dram_pct": dr,
                       "main_tensor_pct": tp}
    print("JSON " + json.dumps(total))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2] if len(sys.argv) > 2 else "tf32")
    else:
        summarise(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "tf32")
