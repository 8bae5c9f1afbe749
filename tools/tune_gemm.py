"""Per-shape GEMM tuner (BASELINE configs[3]: "GEMM shape sweep ... with
per-shape tuned tile parameters, TF32 and BF16"; reference tuner.hpp:560-611).

For every problem of the sweep (the reference grid {64..1024}^3, the squares
2048-8192 and the im2col GEMMs of every VGG16 / ResNet-50 layer -- the rows
of the committed sweep CSV), each precision, the library's own choice
("gemm@<prec>", the cost model) and the tensor-core knobs tile_n x cluster x
K split are timed as device time (CUDA graph of back-to-back column-major nn
calls, median of 3 replays).  All records go to <db>_all.ndjson in the
reference's NDJSON format; the curated DB keeps, per (problem, precision),
the rule's record and the fastest other one only where it wins by >= 5%.
tk_tuning_db_load then applies it on the launch path (tuned_gemm_tile).

    python tools/tune_gemm.py --problems profiles/r01_sweep_tf32.csv \
        --db profiles/r02_tune_gemm.ndjson [--limit-mnk 1e12]
"""
from __future__ import annotations

import argparse
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MIN_GAIN = 0.05
KNOBS = [(0, 0, 0)] + [(n, c, s) for n in (64, 128, 256) for c in (1, 2) for s in (1, 2, 4)]


def config_name(prec, tile_n, cluster, split):
    s = f"gemm@{prec}"
    if tile_n:
        s += f"_n{tile_n}"
    if cluster:
        s += f"_c{cluster}"
    if split == 1:
        s += "_nosplit"
    elif split > 1:
        s += f"_k{split}"
    return s


def problems_from_csv(path):
    out = []
    for line in open(path):
        m = re.match(r"gemm_nn_m(\d+)_n(\d+)_k(\d+),", line)
        if m:
            t = tuple(int(v) for v in m.groups())
            if t not in out:
                out.append(t)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", default="profiles/r01_sweep_tf32.csv")
    ap.add_argument("--db", default="profiles/r02_tune_gemm.ndjson")
    ap.add_argument("--precisions", default="tf32,bf16")
    ap.add_argument("--limit-mnk", type=float, default=2e12, help="skip problems above m*n*k")
    args = ap.parse_args()

    import numpy as np
    import torch
    import paper_1904_05347_b200 as tk
    tk.tuning_db_clear()
    probs = [p for p in problems_from_csv(args.problems) if p[0] * p[1] * p[2] <= args.limit_mnk]
    st = torch.cuda.Stream()
    recs = []
    for (m, n, k) in probs:
        a = torch.rand(m * k, device="cuda") * 2 - 1
        b = torch.rand(k * n, device="cuda") * 2 - 1
        c = torch.empty(m * n, device="cuda")
        shape = tk.GemmShape(m, n, k)
        flops = 2.0 * m * n * k
        for prec in args.precisions.split(","):
            for tn, cl, sp in KNOBS:
                opts = tk.exec_options(prec, tile_n=tn, cluster=cl, split=sp)
                try:
                    with torch.cuda.stream(st):
                        for _ in range(2):
                            tk.gemm_dev(a, b, None, c, shape, None, stream=st, options=opts)
                    st.synchronize()
                except tk.TilekitError:
                    continue
                # back-to-back calls in a graph: ~200 us of work per replay
                est_us = max(flops / 5e8, 2.0)  # ~500 TF/s guess
                reps = int(min(50, max(2, 200 / est_us)))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for _ in range(reps):
                        tk.gemm_dev(a, b, None, c, shape, None, stream=st, options=opts)
                per = []
                with torch.cuda.stream(st):  # replay() launches on the current stream
                    g.replay()
                    st.synchronize()
                    for _ in range(3):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(st)
                        g.replay()
                        e1.record(st)
                        e1.synchronize()
                        per.append(e0.elapsed_time(e1) * 1e6 / reps)  # ns
                del g
                per.sort()
                recs.append({"problem": shape.key(), "config": config_name(prec, tn, cl, sp),
                             "device": "NVIDIA B200", "samples": len(per),
                             "median_ns": int(per[1]), "min_ns": int(per[0]),
                             "mean_ns": int(sum(per) / len(per)), "gflops": flops / per[1],
                             "valid": True, "precision": prec})
        del a, b, c
        torch.cuda.empty_cache()
        print(f"{m}x{n}x{k} done", flush=True)
    all_path = args.db.replace(".ndjson", "_all.ndjson")
    with open(all_path, "w") as fh:
        for r in recs:
            fh.write(json.dumps(r) + "\n")
    groups = {}
    for r in recs:
        groups.setdefault((r["problem"], r["precision"]), []).append(r)
    out, wins = [], []
    for (prob, prec), rs in sorted(groups.items()):
        rule = [r for r in rs if r["config"] == f"gemm@{prec}"]
        best = min(rs, key=lambda r: r["median_ns"])
        if not rule:
            continue
        out.append(rule[0])
        if best is not rule[0] and best["median_ns"] < (1 - MIN_GAIN) * rule[0]["median_ns"]:
            out.append(best)
            wins.append((prob, prec, best["config"], rule[0]["median_ns"] / 1e3, best["median_ns"] / 1e3))
    with open(args.db, "w") as fh:
        for r in out:
            fh.write(json.dumps(r) + "\n")
    for w in wins:
        print(f"{w[0]:34s} {w[1]:5s} {w[2]:28s} rule {w[3]:9.1f} us -> {w[4]:9.1f} us "
              f"({100 * (1 - w[4] / w[3]):.0f}%)")
    print(f"{len(recs)} records, {len(groups)} (problem, precision) groups, {len(wins)} tuned "
          f"choices >= {MIN_GAIN:.0%} over the rules")


if __name__ == "__main__":
    main()
