"""Benchmark: VGG-16 conv stack, NHWC fp32, batch 32 per GPU (BASELINE.json
configs[1]; configs[4] when run on 8 GPUs = batch 256 sharded by batch).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision tf32|fp32]
    python bench.py --impl reference ...     # the reference CPU implementation

--gpus N > 1 outside torchrun re-executes itself under torch.distributed.run
(one process per GPU, NCCL, 127.0.0.1); under torchrun WORLD_SIZE must equal N.
Multi-GPU: rank r owns images [32 r, 32 r + 32) of one
logical batch-(32 N) tensor per layer (each image seeded by its global
index, so the shard is built with no communication), filters are broadcast
once from rank 0 over NCCL; no collective runs inside the timed region.
After timing, one layer's output shards are gathered to rank 0 over NCCL and
compared bitwise with rank 0 recomputing every shard; a GEMM leg (8192^3
TF32, column panels of C = the row-major "M-panels", A broadcast) runs the
same way.

One step = every conv layer of VGG-16 (13 layers, 9 distinct shapes from
proj/data/vgg_layers.csv with the canonical multiplicities) on its own
resident synthetic input, through the C ABI (tk_conv2d_dev).  Metric: total
conv_flops (conv.hpp:19-23; direct-equivalent, the reference's GFLOP/s
convention) / device time.  Timing: CUDA events on the launching stream, L2
flushed (256 MiB write) between steps outside the timed events, max over
ranks.  `e2e` runs the same layers through the host-buffer C ABI
(tk_conv2d_ex) with pinned host buffers: H2D of input+filter and D2H of the
output are inside its timed region.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# (name, H=W, C, K, multiplicity) -- vgg_layers.csv + VGG-16 topology
VGG16 = [
    ("vgg_conv1_1", 224, 3, 64, 1), ("vgg_conv1_2", 224, 64, 64, 1),
    ("vgg_conv2_1", 112, 64, 128, 1), ("vgg_conv2_2", 112, 128, 128, 1),
    ("vgg_conv3_1", 56, 128, 256, 1), ("vgg_conv3_2", 56, 256, 256, 2),
    ("vgg_conv4_1", 28, 256, 512, 1), ("vgg_conv4_2", 28, 512, 512, 2),
    ("vgg_conv5", 14, 512, 512, 3),
]

# ResNet-50 (Caffe variant) conv layers, proj/data/resnet_layers.csv, with the
# multiplicities of the canonical network (53 convs): (name, R, stride, H, C, K, mult)
RESNET50 = [
    ("conv1", 7, 2, 224, 3, 64, 1), ("res2a_branch2a", 1, 1, 56, 64, 64, 1),
    ("res2a_branch2b", 3, 1, 56, 64, 64, 3), ("res2a_branch2c", 1, 1, 56, 64, 256, 3),
    ("res2a_branch1", 1, 1, 56, 64, 256, 1), ("res2b_branch2a", 1, 1, 56, 256, 64, 2),
    ("res3a_branch2a", 1, 2, 56, 256, 128, 1), ("res3a_branch2b", 3, 1, 28, 128, 128, 4),
    ("res3a_branch2c", 1, 1, 28, 128, 512, 4), ("res3a_branch1", 1, 2, 56, 256, 512, 1),
    ("res3b_branch2a", 1, 1, 28, 512, 128, 3), ("res4a_branch2a", 1, 2, 28, 512, 256, 1),
    ("res4a_branch2b", 3, 1, 14, 256, 256, 6), ("res4a_branch2c", 1, 1, 14, 256, 1024, 6),
    ("res4a_branch1", 1, 2, 28, 512, 1024, 1), ("res4b_branch2a", 1, 1, 14, 1024, 256, 5),
    ("res5a_branch2a", 1, 2, 14, 1024, 512, 1), ("res5a_branch2b", 3, 1, 7, 512, 512, 3),
    ("res5a_branch2c", 1, 1, 7, 512, 2048, 3), ("res5a_branch1", 1, 2, 14, 1024, 2048, 1),
    ("res5b_branch2a", 1, 1, 7, 2048, 512, 2),
]

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def plan_str(tk, shape, algo, prec):
    """Compact tk_conv2d_plan_info: kernel/effective precision, CTA group,
    tile, split-K and stream-K tail (e.g. "tc_im2col/tf32 cg2 256x256")."""
    d = tk.conv2d_plan_info(shape, algo, prec)
    s = f"{d['kernel']}/{d['precision']} cg{d['cta_group']} {d['tile_m']}x{d['tile_n']}"
    if d["splits"] > 1:
        s += f" split{d['splits']}"
    if d["tail_pieces"]:
        s += f" tail{d['tail_pieces']}"
    if d["imgs"] > 1:
        s += f" imgs{d['imgs']}"
    if d["flat"]:
        s += " flat"
    if d["precision"] != d["requested_precision"]:
        s += f" (requested {d['requested_precision']})"
    if d.get("tuned"):
        s += " [db]"
    return s


def gemm_plan_str(tk, shape, options):
    """Compact tk_gemm_plan_info (e.g. "tc_plain/tf32 cg2 256x64 A,B in place")."""
    d = tk.gemm_plan_info(shape, options=options)
    s = f"{d['kernel']}/{d['precision']} cg{d['cta_group']} {d['tile_m']}x{d['tile_n']}"
    if d["splits"] > 1:
        s += f" split{d['splits']}"
    if d["tail_pieces"]:
        s += f" tail{d['tail_pieces']}"
    placed = [n for n, f in (("A", d["a_in_place"]), ("B", d["b_in_place"])) if f]
    if d["kernel"] != "exact_simt":
        s += f" {','.join(placed)} in place" if placed else " packed"
    if d.get("tuned"):
        s += " [db]"
    return s


def bound_frac(flops, nbytes, ms, peak_tf, hbm_gbs):
    """Roofline verdict of one layer: HBM-bound when its operational
    intensity (conv_flops / compulsory fp32 bytes) is under the ridge
    peak / HBM; the fraction is then achieved GB/s over HBM, else achieved
    TF/s over the tensor (or FP32) peak."""
    oi = flops / nbytes
    ridge = peak_tf * 1e12 / (hbm_gbs * 1e9)
    if oi < ridge:
        return {"bound": "hbm", "oi": round(oi, 1),
                "frac": round(nbytes / (ms * 1e-3) / 1e9 / hbm_gbs, 3)}
    return {"bound": "tensor", "oi": round(oi, 1),
            "frac": round(flops / (ms * 1e-3) / 1e12 / peak_tf, 3)}


def conv_flops(n, h, c, k):
    return 2 * n * h * h * k * 9 * c


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "bf16", "fp32"])
    ap.add_argument("--batch", type=int, default=32, help="images per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch layer by layer")
    ap.add_argument("--tuning-db", default=",".join(
                        os.path.join(ROOT, "profiles", f) for f in ("r02_tune_ncu.ndjson",
                                                                    "r02_tune_gemm.ndjson")),
                    help="comma-separated NDJSON tuning DBs loaded into the library "
                         "(tools/tune_ncu.py conv plans, tools/tune_gemm.py GEMM tiles); "
                         "'none' = the built-in rules only")
    ap.add_argument("--no-multi", action="store_true",
                    help="skip the multi-GPU verification gather and the GEMM column-panel leg "
                         "(profiling runs: the step's launches are then the last ones)")
    ap.add_argument("--no-layers", action="store_true",
                    help="skip the per-layer kernel timing (profiling runs: the step's launches "
                         "are then the last ones after the L2 flush)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md)
# ---------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("BENCH_SMI_MS", "20")], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:  # sampler is live
                time.sleep(0.01)
            self.lines.clear()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the unmodified reference on the host cores
# ---------------------------------------------------------------------------
# The reference's fastest CPU algorithm per VGG-16 layer (its own conv2d
# selector), from timing all of naive/tiled/im2col/winograd on the host.
REF_ALGO = {
    "vgg_conv1_1": "tiled_t4x5_v4x2", "vgg_conv1_2": "winograd_t4x4",
    "vgg_conv2_1": "winograd_t4x4", "vgg_conv2_2": "winograd_t4x4",
    "vgg_conv3_1": "winograd_t4x4", "vgg_conv3_2": "winograd_t2x2",
    "vgg_conv4_1": "winograd_t4x4", "vgg_conv4_2": "winograd_t2x2",
    "vgg_conv5": "winograd_t2x2",
}


def vgg_instances():
    out = []
    for name, h, c, k, mult in VGG16:
        out += [(name, h, c, k)] * mult
    return out


class CpuReference:
    """Times the reference's own conv2d on host cores: oracle/_ref (the
    unmodified reference headers behind ref_shim.cpp) when it was built in
    this tree, else the C restatement (kind "port").  A sample is one VGG-16
    layer instance at batch 1 (1/32 of that layer's per-GPU work)."""

    def __init__(self):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle as O
        O.build()
        self.O = O
        self.cores = os.cpu_count() or 1
        os.environ["TILEKIT_THREADS"] = str(self.cores)
        self.kind = "reference" if O.have_ref() else "port"
        self.cache = {}

    def layer(self, name, h, c, k):
        O = self.O
        if name not in self.cache:
            s = O.Conv(1, h, h, c, k, 3, 3, 1, True)
            x = O.fill_random(int(np.prod(s.in_shape)), 1).reshape(s.in_shape)
            f = O.fill_random(int(np.prod(s.filt_shape)), 2).reshape(s.filt_shape)
            self.cache[name] = (s, x, f)
        s, x, f = self.cache[name]
        algo = REF_ALGO[name]
        t0 = time.perf_counter()
        if self.kind == "reference":
            O.ref_conv2d(s, algo, x, f)
        elif algo.startswith("winograd"):
            O.conv2d_winograd(s, int(algo[-1]), x, f)
        else:
            O.conv2d_naive(s, x, f)
        return s.flops(), time.perf_counter() - t0

    def full_pass(self):
        fl, sec = 0, 0.0
        for inst in vgg_instances():
            a, b = self.layer(*inst)
            fl += a
            sec += b
        return fl, sec


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref = CpuReference()
    # A step = one full VGG16 stack (all 13 layer instances) at batch 1: the
    # same per-layer mix as the GPU step, 1/32 of its images (~0.7 s on 16
    # host threads), so the value does not depend on K.
    for _ in range(max(1, min(args.warmup, 2))):
        ref.full_pass()
    fl, sec = 0, 0.0
    for _ in range(args.steps):
        a, b = ref.full_pass()
        fl += a
        sec += b
    value = fl / sec / 1e9
    line = {
        "impl": "reference", "metric": "VGG16 conv-stack GFLOP/s (conv_flops / time)",
        "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * sec / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (fill_random, tuner.hpp:293-297)",
        "config": {"workload": "VGG16 13 conv layers (3x3/s1/Same, NHWC fp32); each step one "
                               "full 13-layer pass at batch 1 (bounded CPU sample of the "
                               "batch-32 GPU workload)",
                   "algorithms": REF_ALGO},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": ref.cores,
                         "kind": ref.kind,
                         "sample": f"{args.steps} full VGG16 passes at batch 1, reference "
                                   "conv2d with its fastest CPU algorithm per layer"},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def relaunch(args) -> int:
    """--gpus N outside torchrun: re-execute this script under
    torch.distributed.run with N local ranks (rank 0 prints the line)."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}),
              flush=True)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)

    import torch
    import torch.distributed as dist
    import paper_1904_05347_b200 as tk
    from paper_1904_05347_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    N = args.batch
    prec = args.precision
    lo_img, hi_img = rank * N, (rank + 1) * N  # this rank's images of the global batch
    # The tuner's DB (lookup_best on the launch path): calls with automatic
    # knobs take the fastest recorded knobs of their shape.
    db_records = 0
    db_paths = [] if args.tuning_db == "none" else \
        [p_ for p_ in args.tuning_db.split(",") if p_ and os.path.exists(p_)]
    for p_ in db_paths:
        db_records += tk.tuning_db_load(p_)

    # Resident inputs: one independent seeded input + filter per layer
    # instance (the reference `layers` harness, tilekit_cli.cpp:374-403).
    # Inputs: this rank's slice of the logical batch-(N * world) tensor;
    # filters: seeded on rank 0, replicated by one NCCL broadcast.
    gen = torch.Generator(device=dev).manual_seed(1234)
    layers = []
    for name, h, c, k, mult in VGG16:
        for rep in range(mult):
            shape = tk.ConvShape(N, h, h, c, k, 3, 3, 1, True)
            algo = tk.parse_conv_params("im2col")
            x = shard.seeded_images((h, h, c), lo_img, hi_img, 1234, len(layers), dev)
            f = torch.rand((3, 3, c, k), device=dev, generator=gen) * 2 - 1
            shard.broadcast_(f)
            y = torch.empty((N, h, h, k), device=dev)
            ws_n = tk.conv2d_workspace_size(shape, algo, prec)
            ws = torch.empty(max(ws_n, 4) // 4 + 1, device=dev)
            layers.append(dict(name=name, shape=shape, algo=algo, x=x, f=f, y=y, ws=ws,
                               flops=conv_flops(N, h, c, k), hwc=(h, h, c)))
    flush = torch.empty(64 * 1024 * 1024, device=dev)  # 256 MiB > 126 MB L2
    step_flops = sum(L["flops"] for L in layers)

    def step():
        for L in layers:
            tk.conv2d_dev(L["x"], L["f"], L["y"], L["shape"], L["algo"], precision=prec,
                          workspace=L["ws"], stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # The step is captured once as a CUDA graph (launch-bound inner loop:
    # 26 launches whose host-side setup would otherwise gate the small
    # layers); kernel parameters, TMA descriptors included, are captured by
    # value.  gpu_launches counts the kernels inside the graph.
    graph = None
    launches_per_step = None
    # Per-layer device time inside the timed steps: timing event-record nodes
    # in the step graph between consecutive layer launches on the main stream.
    in_step_events = not args.no_graph and os.environ.get("BENCH_STEP_EVENTS", "0") == "1"
    lay_ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(layers) + 1)]
    in_step = np.zeros(len(layers))
    if not args.no_graph:
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(stream)
        l0 = tk.launch_count()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        with torch.cuda.graph(graph, stream=cap):
            # Filter-side work (prepare: tensor-core filter repack) depends only
            # on the filters: fork it to a side stream so it overlaps earlier
            # layers; each layer's run joins on its own prepare.
            side.wait_stream(cap)
            ready = []
            with torch.cuda.stream(side):
                for L in layers:
                    tk.conv2d_prepare_dev(L["f"], L["shape"], L["algo"], L["ws"], precision=prec,
                                          stream=side)
                    ev = torch.cuda.Event()
                    ev.record(side)
                    ready.append(ev)
            for i, (L, ev) in enumerate(zip(layers, ready)):
                cap.wait_event(ev)
                if in_step_events:
                    lay_ev[i].record(cap)
                tk.conv2d_run_dev(L["x"], L["f"], L["y"], L["shape"], L["algo"], L["ws"],
                                  precision=prec, stream=cap)
            if in_step_events:
                lay_ev[-1].record(cap)
            cap.wait_stream(side)
        launches_per_step = tk.launch_count() - l0
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            step()

    # Timed steps.
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = tk.launch_count()
    times = []
    extra_steps = 0
    step_flush = os.environ.get("BENCH_STEP_FLUSH", "1") == "1"
    # A ~0.5 ms GPU spin before each step's start event (outside the timed
    # region): the host has queued the step graph before the GPU reaches the
    # event, so the events time the step and not host-side submission
    # jitter (measured: without it 1-in-5 steps carried a 0.1-0.2 ms idle
    # gap, mean 1.52 vs median 1.475 ms; with it mean 1.473, max 1.50 ms).
    prespin = int(os.environ.get("BENCH_PRESPIN", "1000000"))
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            if step_flush:
                flush.zero_()
            if prespin:
                torch.cuda._sleep(prespin)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            if in_step_events:
                in_step += [lay_ev[i].elapsed_time(lay_ev[i + 1]) for i in range(len(layers))]
        timed_samples = len(clocks.lines)
        launches = tk.launch_count() - launches0
        # A short timed region (small --steps) can end between two 20 ms
        # samples: keep the same step running, untimed, until three samples
        # under this load exist (reported as samples_after_timed).
        t_end = time.time() + 2.0
        while len(clocks.lines) < 3 and clocks.proc is not None and time.time() < t_end:
            flush.zero_()
            run_step()
            torch.cuda.synchronize()
            extra_steps += 1
    if launches_per_step is not None:
        launches = launches_per_step * args.steps
    torch.cuda.synchronize()
    rank_ms = shard.all_gather_scalar(float(sum(times)) / args.steps, device=dev)
    total_ms = shard.max_over_ranks(float(sum(times)), device=dev)
    ms_per_step = total_ms / args.steps
    value = step_flops * world / (ms_per_step * 1e-3) / 1e9

    # Multi-GPU verification (outside every timed region): the last layer's
    # output shards (vgg_conv5, 12.8 MB per rank) gathered to rank 0 over
    # NCCL, compared bitwise with rank 0 recomputing each shard from its
    # seeded images (same shape, same plan => same bits), and image 0 of each
    # shard against the library's bit-exact FP32 path.
    multi = {"ranks": world, "rank_ms_per_step": [round(v, 4) for v in rank_ms],
             "images_per_rank": N, "global_batch": N * world}
    vi = len(layers) - 1
    Lv = layers[vi]
    torch.cuda.synchronize()
    parts = shard.gather_to(Lv["y"], 0) if not args.no_multi else []
    if rank == 0 and not args.no_multi:
        same, worst = True, 0.0
        for r, part in enumerate(parts):
            xr = shard.seeded_images(Lv["hwc"], r * N, (r + 1) * N, 1234, vi, dev)
            yr = torch.empty_like(Lv["y"])
            tk.conv2d_dev(xr, Lv["f"], yr, Lv["shape"], Lv["algo"], precision=prec, stream=stream)
            s1 = tk.ConvShape(1, *Lv["hwc"][:2], Lv["hwc"][2], Lv["shape"].features, 3, 3, 1, True)
            ye = torch.empty((1,) + tuple(Lv["y"].shape[1:]), device=dev)
            tk.conv2d_dev(xr[:1].contiguous(), Lv["f"], ye, s1, Lv["algo"], precision="fp32",
                          stream=stream)
            torch.cuda.synchronize()
            same &= bool(torch.equal(yr.view(torch.int32), part.view(torch.int32)))
            worst = max(worst, float((part[:1] - ye).abs().max() / ye.abs().max().clamp_min(1e-6)))
        multi["verify"] = {"layer": Lv["name"], "gathered_bytes": int(Lv["y"].numel() * 4 * world),
                           "shards_bitwise_equal_to_recompute": same,
                           "max_scaled_error_vs_fp32_exact_img0": worst}
    del parts

    # GEMM leg (BASELINE configs[3] at 8192^3, TF32): column panels of the
    # column-major C (the row-major formulation's M-panels), panel edges on
    # the 256-wide tensor-core tile, A replicated by broadcast, each rank's
    # B panel seeded per 256-column block.  Strong scaling: fixed total work.
    if not args.no_multi:
        gn = 8192
        glo, ghi = shard.panel_range(gn, world, rank, 256)
        ga = torch.rand(gn * gn, device=dev, generator=torch.Generator(device=dev).manual_seed(99)) * 2 - 1
        shard.broadcast_(ga)
        gb = shard.seeded_columns(gn, glo, ghi, 4242, 256, dev)
        gc = torch.empty(gn * (ghi - glo), device=dev)
        gshape = tk.GemmShape(gn, ghi - glo, gn)
        for _ in range(2):
            tk.gemm_dev(ga, gb, None, gc, gshape, None, precision="tf32", stream=stream)
        gts = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(5):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            tk.gemm_dev(ga, gb, None, gc, gshape, None, precision="tf32", stream=stream)
            b_.record(stream)
            b_.synchronize()
            gts.append(a_.elapsed_time(b_))
        g_ms = float(np.median(gts))
        g_rank = shard.all_gather_scalar(g_ms, device=dev)
        g_max = max(g_rank)
        panels = {"value": round(2 * gn ** 3 / (g_max * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
                  "scaling": "strong", "ms_max_over_ranks": round(g_max, 4),
                  "rank_ms": [round(v, 4) for v in g_rank], "panel_cols": ghi - glo,
                  "config": f"C = A B, {gn}^3 TF32, column panels of C (A broadcast)"}
        gparts = shard.gather_to(gc[: gn * 256].clone(), 0)  # first 256 columns of every panel
        if rank == 0:
            same = True
            for r, part in enumerate(gparts):
                rlo, rhi = shard.panel_range(gn, world, r, 256)
                br = shard.seeded_columns(gn, rlo, rhi, 4242, 256, dev)
                cr = torch.empty(gn * (rhi - rlo), device=dev)
                tk.gemm_dev(ga, br, None, cr, tk.GemmShape(gn, rhi - rlo, gn), None, precision="tf32",
                            stream=stream)
                torch.cuda.synchronize()
                same &= bool(torch.equal(cr[: gn * 256].view(torch.int32), part.view(torch.int32)))
                del br, cr
            panels["verify_first_256_cols_bitwise"] = same
        multi["gemm8192_tf32_panels"] = panels
        del ga, gb, gc, gparts

    # Per-layer device times of the conv kernels (after the timed steps; same
    # stream, CUDA events),
    # for the roofline.  With graphs: one graph replays R x [L2 eviction, the
    # layer's run phase] and a second R x [L2 eviction]; the layer's kernel time
    # is their difference / R -- L2-cold like the step, without the graph
    # launch latency (~4-6 us) that an event pair around one replay adds.
    # The filter prepare (tiny, overlapped in the step) is not included.
    per_layer = []
    reps = 4

    def timed(fn, n=3, pre=None):
        ts = []
        for _ in range(n):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            if pre is not None:
                pre()
            torch.cuda.synchronize()
            ev[0].record(stream)
            fn()
            ev[1].record(stream)
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        return float(np.median(ts))

    # The per-layer eviction reads the 256 MiB buffer (clean lines): a write
    # flush would leave ~126 MB of dirty lines whose write-back then lands on
    # the timed layer.
    flush_sink = torch.empty((), device=dev)

    evict_read = os.environ.get("BENCH_EVICT", "read") == "read"

    def evict():
        if evict_read:
            torch.sum(flush, dim=0, out=flush_sink)
        else:
            flush.zero_()

    flush_ms = None
    if not args.no_graph:
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(stream)
        fg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(fg, stream=cap):
            for _ in range(reps):
                evict()
        with torch.cuda.stream(stream):
            flush_ms = timed(fg.replay)

    def kernel_ms(run_on):
        """Device time of run_on(stream) (a prepared layer's run phase),
        L2-cold, without launch latency (graph of reps x [flush, run])."""
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(stream)
        lg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(lg, stream=cap):
            for _ in range(reps):
                evict()
                run_on(cap)
        with torch.cuda.stream(stream):
            return max(timed(lg.replay) - flush_ms, 1e-6) / reps

    for L in ([] if args.no_layers else layers):
        if not args.no_graph:
            per_layer.append(kernel_ms(
                lambda st, L=L: tk.conv2d_run_dev(L["x"], L["f"], L["y"], L["shape"], L["algo"],
                                                  L["ws"], precision=prec, stream=st)))
        else:
            def one(L=L):
                tk.conv2d_dev(L["x"], L["f"], L["y"], L["shape"], L["algo"], precision=prec,
                              workspace=L["ws"], stream=stream)
            per_layer.append(timed(one, pre=evict))


    # End-to-end through the host-buffer C ABI (pinned host memory).
    e2e = None
    if not args.no_e2e:
        host = []
        pinned = [True]

        def host_buf(t):
            # Page-locked when the host allows it (both copy directions then
            # overlap); pageable otherwise, recorded in the e2e entry.
            try:
                return t.pin_memory().numpy()
            except RuntimeError:
                pinned[0] = False
                return t.numpy()

        for L in layers:
            if L["name"] in [h["name"] for h in host]:
                continue
            host.append(dict(name=L["name"], shape=L["shape"], algo=L["algo"],
                             x=host_buf(L["x"].cpu()), f=host_buf(L["f"].cpu()),
                             y=host_buf(torch.empty(tuple(L["y"].shape)))))
        by_name = {h["name"]: h for h in host}
        seq = [by_name[L["name"]] for L in layers]
        h2d = sum(h["x"].nbytes + h["f"].nbytes for h in seq)
        d2h = sum(h["y"].nbytes for h in seq)
        for h in seq:  # warm the pool allocator
            out = tk.conv2d(h["x"], h["f"], h["shape"], h["algo"], precision=prec)
        e2e_steps = max(1, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            for h in seq:
                lib = tk.lib()
                rc = lib.tk_conv2d_ex(ctypes.byref(h["shape"].c()), ctypes.byref(h["algo"].c()),
                                      ctypes.byref(tk.exec_options(prec)),
                                      h["x"].ctypes.data_as(ctypes.c_void_p),
                                      h["f"].ctypes.data_as(ctypes.c_void_p),
                                      h["y"].ctypes.data_as(ctypes.c_void_p))
                tk._check(rc)
        e2e_s = shard.max_over_ranks((time.perf_counter() - t0) / e2e_steps, device=dev)
        e2e = {"value": round(step_flops * world / e2e_s / 1e9, 2), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(e2e_s * 1e3, 3), "api": "tk_conv2d_ex (host buffers)",
               "host_memory": "pinned" if pinned[0] else "pageable"}

    peaks, peaks_kind = load_peaks()
    # Dominant kernel: the implicit-GEMM conv (tc_gemm_kernel) -- its share
    # is the whole step except the tiny filter-pack launches.
    # Per-layer times inside the timed steps (event nodes in the step graph,
    # averaged over the K steps) when available, else the isolated kernels.
    step_layer = list(in_step / max(1, args.steps)) if in_step_events else list(per_layer)
    if not step_layer:  # --no-layers: the step itself
        step_layer = [ms_per_step * L["flops"] / step_flops for L in layers]
        per_layer = list(step_layer)
    lay_ms = float(sum(step_layer))
    achieved_tf = step_flops / (lay_ms * 1e-3) / 1e12
    if prec == "bf16":
        peak_tf = peaks["bf16_tflops"]
        peak_note = f"{peaks_kind} bf16 burst {peaks['bf16_tflops']} TF/s"
    elif prec == "tf32":
        peak_tf = peaks["bf16_tflops"] / 2.0
        peak_note = f"TF32 = 1/2 of {peaks_kind} bf16 burst {peaks['bf16_tflops']} TF/s"
    else:
        peak_tf = 148 * 128 * 2 * 1.965e9 / 1e12 / 2
        peak_note = "FP32 exact FMUL+FADD cap = 1/2 of 74.4 TF/s FFMA"
    # DRAM traffic of the dominant kernel per step, from the committed ncu
    # launch list of this same command (profiles/, tools/launch_summary.py),
    # next to the compulsory bytes of the step (each layer's input, filter
    # and output once, conv_oi's model).
    traffic, traffic_src = None, None
    import glob
    profs = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_launches_{prec}.json")))  # newest round
    prof = profs[-1] if profs else ""
    if prof:
        kern = json.load(open(prof))["kernels"]
        tb = sum(v["dram_bytes"] for k, v in kern.items()
                 if any(x in k for x in ("tc_gemm_kernel", "exact_gemm", "tail_reduce",
                                         "splitk_reduce", "pad_phase", "to_bf16")))
        traffic, traffic_src = int(tb), os.path.relpath(prof, ROOT)
    compulsory = sum(4 * (L["x"].numel() + L["f"].numel() + L["y"].numel()) for L in layers)
    roofline = {"bound": "tensor", "achieved": round(achieved_tf, 2), "peak": round(peak_tf, 1),
                "unit": "TFLOP/s", "frac": round(achieved_tf / peak_tf, 4), "traffic": traffic,
                "traffic_unit": "DRAM bytes per step, all conv-path launches excl. the overlapped filter packs (ncu dram__bytes_read+write)",
                "traffic_source": traffic_src, "compulsory_bytes": int(compulsory),
                "kernel": "exact_gemm_loc_kernel" if prec == "fp32" else "tc_gemm_kernel (implicit-GEMM conv)",
                "peak_source": peak_note}

    layer_rows = []
    for L, ms, kms in zip(layers, step_layer, per_layer):
        nbytes = 4 * (L["x"].numel() + L["f"].numel() + L["y"].numel())
        layer_rows.append(dict({"layer": L["name"], "ms": round(ms, 4), "kernel_ms": round(kms, 4),
                                "tflops": round(L["flops"] / (ms * 1e-3) / 1e12, 2),
                                "plan": plan_str(tk, L["shape"], L["algo"], prec)},
                               **bound_frac(L["flops"], nbytes, ms, peak_tf, peaks["hbm_gbs"])))

    peaks, peaks_kind = load_peaks()
    # Secondary lines (same run, same resident inputs): the other precisions
    # of the stack and BASELINE configs[0], SGEMM 1024^3 (row-major C = A B as
    # the column-major nn call with operands swapped).
    secondary = {}
    if not args.no_secondary and world == 1:
        def stack_ms(p_, reps):
            ts = []
            for _ in range(reps):
                flush.zero_()
                if prespin:
                    torch.cuda._sleep(prespin)  # (see the timed steps)
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                for L in layers:
                    tk.conv2d_dev(L["x"], L["f"], L["y"], L["shape"], L["algo"], precision=p_,
                                  workspace=None, stream=stream)
                b_.record(stream)
                b_.synchronize()
                ts.append(a_.elapsed_time(b_))
            return float(np.median(ts))
        for p_ in [q for q in ("tf32", "bf16", "3xtf32", "fp32") if q != prec]:
            stack_ms(p_, 1)
            ms = stack_ms(p_, 3 if p_ != "fp32" else 1)
            secondary[f"vgg16_{p_}"] = {"value": round(step_flops / (ms * 1e-3) / 1e9, 1),
                                         "unit": "GFLOP/s", "ms_per_step": round(ms, 3),
                                         "bit_exact": p_ == "fp32"}
        # BF16 with bf16 activations in HBM (tk_exec_options.io = bf16): each
        # layer reads a bf16 input and writes a bf16 output -- a BF16
        # network's layer-to-layer format (the producing layer's epilogue
        # writes what the next one reads), so no fp32 -> bf16 conversion pass
        # and half the output bytes.  Same layers, filters and per-call
        # filter pack as vgg16_bf16.
        io_opts = tk.exec_options("bf16", io="bf16")
        xb_ = [L["x"].to(torch.bfloat16) for L in layers]
        yb_ = [torch.empty(tuple(L["y"].shape), device=dev, dtype=torch.bfloat16) for L in layers]

        def stack_io_ms(reps):
            ts = []
            for _ in range(reps):
                flush.zero_()
                if prespin:
                    torch.cuda._sleep(prespin)  # (see the timed steps)
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                for L, xb, yb in zip(layers, xb_, yb_):
                    tk.conv2d_dev(xb, L["f"], yb, L["shape"], L["algo"], workspace=None,
                                  stream=stream, options=io_opts)
                b_.record(stream)
                b_.synchronize()
                ts.append(a_.elapsed_time(b_))
            return float(np.median(ts))
        stack_io_ms(1)
        ms = stack_io_ms(3)
        secondary["vgg16_bf16_io"] = {"value": round(step_flops / (ms * 1e-3) / 1e9, 1),
                                      "unit": "GFLOP/s", "ms_per_step": round(ms, 3),
                                      "activations": "bf16 in / bf16 out (tk_exec_options.io)"}
        del xb_, yb_
        # BASELINE configs[1] at batch 1: the 13 VGG16 layers on one image
        # (latency-bound: 13 launches of small grids), TF32, as one graph.
        b1 = []
        for name, hh, cc, kk, mult in VGG16:
            shp = tk.ConvShape(1, hh, hh, cc, kk, 3, 3, 1, True)
            for _ in range(mult):
                b1.append((shp, torch.rand(shp.in_shape, device=dev, generator=gen) * 2 - 1,
                           torch.rand(shp.filt_shape, device=dev, generator=gen) * 2 - 1,
                           torch.empty(shp.out_shape, device=dev),
                           torch.empty(tk.conv2d_workspace_size(shp, tk.parse_conv_params("im2col"),
                                                                prec) // 4 + 1, device=dev)))
        b1_flops = sum(shp.flops() for shp, *_ in b1)

        def b1_pass(st_):
            for shp, x, f, y, ws in b1:
                tk.conv2d_dev(x, f, y, shp, tk.parse_conv_params("im2col"), precision=prec,
                              workspace=ws, stream=st_)
        b1_pass(stream)
        torch.cuda.synchronize()
        g_b1 = None
        if not args.no_graph:
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(stream)
            g_b1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_b1, stream=cap):
                b1_pass(cap)
            g_b1.replay()
            torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            if prespin:
                torch.cuda._sleep(prespin)  # (see the timed steps)
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            if g_b1 is not None:
                g_b1.replay()
            else:
                b1_pass(stream)
            b_.record(stream)
            b_.synchronize()
            ts.append(a_.elapsed_time(b_))
        ms = float(np.median(ts))
        secondary[f"vgg16_batch1_{prec}"] = {"value": round(b1_flops / (ms * 1e-3) / 1e9, 1),
                                             "unit": "GFLOP/s", "ms_per_step": round(ms, 4),
                                             "note": "L2-warm (inputs fit in L2)"}

        # BASELINE configs[2]: ResNet-50 conv stack (53 layers) at batch 32.
        rn = []
        for name, r, stv, h, c, k, mult in RESNET50:
            shp = tk.ConvShape(N, h, h, c, k, r, r, stv, True)
            x = torch.rand((N, h, h, c), device=dev, generator=gen) * 2 - 1
            f = torch.rand((r, r, c, k), device=dev, generator=gen) * 2 - 1
            y = torch.empty(shp.out_shape, device=dev)
            ws = torch.empty(tk.conv2d_workspace_size(shp, tk.parse_conv_params("im2col"), prec)
                             // 4 + 1, device=dev)
            rn.append((shp, x, f, y, ws, mult, shp.flops()))
        rn_flops = sum(fl * m for *_, m, fl in rn)
        im2col = tk.parse_conv_params("im2col")
        for p_ in ("tf32", "bf16", "bf16_io"):
            # One workspace per layer instance (each of a shape's `mult`
            # instances is its own layer with its own prepared filter).
            # bf16_io: BF16 with bf16 activations in HBM (see vgg16_bf16_io).
            io_ = p_ == "bf16_io"
            o_ = tk.exec_options("bf16" if io_ else p_, io="bf16" if io_ else "fp32")
            inst = [(shp, x.to(torch.bfloat16) if io_ else x, f,
                     torch.empty(tuple(y.shape), device=dev, dtype=torch.bfloat16) if io_ else y,
                     torch.empty(tk.conv2d_workspace_size(shp, im2col, options=o_) // 4 + 1,
                                 device=dev))
                    for shp, x, f, y, _, mult, _ in rn for _ in range(mult)]

            def rn_pass(s_main, s_side):
                # As the VGG step: filter prepares forked to a side stream,
                # each run joins on its own prepare.
                s_side.wait_stream(s_main)
                ready = []
                with torch.cuda.stream(s_side):
                    for shp, x, f, y, ws in inst:
                        tk.conv2d_prepare_dev(f, shp, im2col, ws, options=o_, stream=s_side)
                        ev = torch.cuda.Event()
                        ev.record(s_side)
                        ready.append(ev)
                for (shp, x, f, y, ws), ev in zip(inst, ready):
                    s_main.wait_event(ev)
                    tk.conv2d_run_dev(x, f, y, shp, im2col, ws, options=o_, stream=s_main)
                s_main.wait_stream(s_side)
            side_rn = torch.cuda.Stream(device=dev)
            rn_pass(stream, side_rn)
            torch.cuda.synchronize()
            g_rn = None
            if not args.no_graph:
                cap = torch.cuda.Stream(device=dev)
                cap.wait_stream(stream)
                g_rn = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_rn, stream=cap):
                    rn_pass(cap, side_rn)
                g_rn.replay()
                torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                flush.zero_()
                if prespin:
                    torch.cuda._sleep(prespin)  # (see the timed steps)
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                if g_rn is not None:
                    g_rn.replay()
                else:
                    rn_pass(stream, side_rn)
                b_.record(stream)
                b_.synchronize()
                ts.append(a_.elapsed_time(b_))
            ms = float(np.median(ts))
            secondary[f"resnet50_{p_}"] = {"value": round(rn_flops / (ms * 1e-3) / 1e9, 1),
                                            "unit": "GFLOP/s", "ms_per_step": round(ms, 3),
                                            "step_gflop": round(rn_flops / 1e9, 2),
                                            "batch_per_gpu": N}
            if io_:
                secondary[f"resnet50_{p_}"]["activations"] = "bf16 in / bf16 out (tk_exec_options.io)"
            if not args.no_graph and p_ == prec:
                # Kernel time per distinct layer shape (first instance, its
                # filter prepared by the pass above), as the VGG layers.
                pk = peaks["bf16_tflops"] / (2.0 if p_ == "tf32" else 1.0)
                rows, k0 = [], 0
                for (name, *_rest), (shp, x, f, y, ws, mult, fl) in zip(RESNET50, rn):
                    _, _, _, _, ws0 = inst[k0]
                    k0 += mult
                    kms = kernel_ms(lambda st, shp=shp, x=x, f=f, y=y, ws0=ws0: tk.conv2d_run_dev(
                        x, f, y, shp, im2col, ws0, precision=p_, stream=st))
                    nbytes = 4 * (x.numel() + f.numel() + y.numel())
                    rows.append(dict({"layer": name, "ms": round(kms, 4),
                                      "tflops": round(fl / (kms * 1e-3) / 1e12, 1),
                                      "frac_of_peak": round(fl / (kms * 1e-3) / 1e12 / pk, 3),
                                      "plan": plan_str(tk, shp, im2col, p_)},
                                     **bound_frac(fl, nbytes, kms, pk, peaks["hbm_gbs"])))
                secondary[f"resnet50_{p_}"]["layers"] = rows
        # configs[2]'s "tiled path": the whole 53-layer stack through the
        # exact FP32 tiled algorithm (bit-identical to the reference).
        tiled = tk.parse_conv_params("tiled_t2x2_v4x8")  # 2x2-pixel patches x 8 features

        def rn_tiled(st_):
            for shp, x, f, y, ws, mult, _fl in rn:
                for _ in range(mult):
                    tk.conv2d_dev(x, f, y, shp, tiled, precision="fp32", stream=st_)
        rn_tiled(stream)
        torch.cuda.synchronize()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        if prespin:
            torch.cuda._sleep(prespin)
        a_.record(stream)
        rn_tiled(stream)
        b_.record(stream)
        b_.synchronize()
        ms = a_.elapsed_time(b_)
        secondary["resnet50_tiled_fp32"] = {"value": round(rn_flops / (ms * 1e-3) / 1e9, 1),
                                            "unit": "GFLOP/s", "ms_per_step": round(ms, 3),
                                            "algorithm": "tiled_t2x2_v4x8", "bit_exact": True}
        del rn
        # BASELINE configs[1]'s algorithm comparison: every distinct VGG16
        # layer at batch 32 through each conv algorithm of the selector
        # (direct / tiled / im2col are one exact-FP32 kernel -- the same
        # ascending (x, y, c) sum -- so "tiled" stands for them; im2col and
        # Winograd F(2x2) / F(4x4) on the tensor cores in TF32, Winograd F(2x2)
        # also exact FP32).  Whole conv2d_dev calls (filter transform
        # included, as the reference's conv2d does) from a graph, L2-cold,
        # launch latency removed as for the layers.  GFLOP/s count the
        # direct-equivalent conv_flops for every algorithm (tuner.hpp:442).
        # Batch 1 too (configs[1] names "batch 1 and 32"): there the layers
        # are latency-bound small grids.
        for nb in ((N, 1) if not args.no_graph else ()):
            algos = [("naive_fp32", "naive", "fp32"), ("tiled_fp32", "tiled_t2x2_v4x8", "fp32"),
                     ("tiled_t4x5_v4x2_fp32", "tiled_t4x5_v4x2", "fp32"),
                     ("im2col_tf32", "im2col", "tf32"), ("im2col_bf16", "im2col", "bf16"),
                     ("winograd_t2x2_tf32", "winograd_t2x2", "tf32"),
                     ("winograd_t4x4_tf32", "winograd_t4x4", "tf32"),
                     ("winograd_t2x2_fp32", "winograd_t2x2", "fp32")]
            table = {}
            for name, h, c, k, _mult in VGG16:
                shp = tk.ConvShape(nb, h, h, c, k, 3, 3, 1, True)
                x = torch.rand((nb, h, h, c), device=dev, generator=gen) * 2 - 1
                f = torch.rand((3, 3, c, k), device=dev, generator=gen) * 2 - 1
                y = torch.empty(shp.out_shape, device=dev)
                row = {}
                for key, algo_name, p_ in algos:
                    algo = tk.parse_conv_params(algo_name)
                    try:
                        wsz = tk.conv2d_workspace_size(shp, algo, p_)
                    except tk.TilekitError:
                        continue
                    ws = torch.empty(max(wsz, 4) // 4 + 1, device=dev)
                    run = (lambda st, algo=algo, p_=p_, ws=ws: tk.conv2d_dev(
                        x, f, y, shp, algo, precision=p_, workspace=ws, stream=st))
                    run(stream)  # warm (allocator, descriptors)
                    torch.cuda.synchronize()
                    ms = kernel_ms(run)
                    row[key] = {"ms": round(ms, 4),
                                "gflops": round(shp.flops() / (ms * 1e-3) / 1e9, 1)}
                    del ws
                table[name] = row
                del x, f, y
            secondary[f"vgg16_algorithms_b{nb}"] = table
        # BASELINE configs[3]: large square GEMMs on the tensor cores
        # (column-major nn through tk_gemm_dev; operands in HBM, > L2 from 4096;
        # the fp32-operand BF16 calls include their two operand packs).
        # value/ms: device time of back-to-back calls (graph replay);
        # api_ms: one call between events, host work included.
        for n in (2048, 4096, 8192):
            ga = torch.rand(n * n, device=dev) * 2 - 1
            gb = torch.rand(n * n, device=dev) * 2 - 1
            gc = torch.empty(n * n, device=dev)
            gshape = tk.GemmShape(n, n, n)
            for p_ in ("tf32", "bf16", "bf16_io", "3xtf32"):
                if p_ == "3xtf32" and n != 8192:
                    continue
                # bf16_io: bf16 operands in HBM (exec_options io="in_bf16"),
                # the fp32 -> bf16 conversion of A and B not in the timed call
                io_ = p_ == "bf16_io"
                o_ = tk.exec_options("bf16" if io_ else p_, io="in_bf16" if io_ else "fp32")
                ga_, gb_ = (ga.to(torch.bfloat16), gb.to(torch.bfloat16)) if io_ else (ga, gb)
                for _ in range(2):
                    tk.gemm_dev(ga_, gb_, None, gc, gshape, None, stream=stream, options=o_)
                ts = []
                for _ in range(5):
                    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a_.record(stream)
                    tk.gemm_dev(ga_, gb_, None, gc, gshape, None, stream=stream, options=o_)
                    b_.record(stream)
                    b_.synchronize()
                    ts.append(a_.elapsed_time(b_))
                api_ms = float(np.median(ts))
                # Device time without the host work of each call (as for
                # SGEMM 1024^3): R back-to-back calls captured in a graph,
                # median of 3 replays.
                R = {2048: 10, 4096: 5, 8192: 2}[n]
                cap = torch.cuda.Stream(device=dev)
                cap.wait_stream(stream)
                gg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gg, stream=cap):
                    for _ in range(R):
                        tk.gemm_dev(ga_, gb_, None, gc, gshape, None, stream=cap, options=o_)
                gg.replay()
                torch.cuda.synchronize()
                reps_ = []
                for _ in range(3):
                    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a_.record(stream)
                    gg.replay()
                    b_.record(stream)
                    b_.synchronize()
                    reps_.append(a_.elapsed_time(b_) / R)
                del gg
                ms = float(np.median(reps_))
                tf = 2 * n ** 3 / (ms * 1e-3) / 1e12
                pk = peaks["bf16_tflops"] / {"tf32": 2.0, "bf16": 1.0, "bf16_io": 1.0, "3xtf32": 6.0}[p_]
                secondary[f"gemm{n}_{p_}"] = {"value": round(tf * 1e3, 1), "unit": "GFLOP/s",
                                              "ms": round(ms, 4), "frac_of_peak": round(tf / pk, 4),
                                              "api_ms": round(api_ms, 4),
                                              "plan": gemm_plan_str(tk, gshape, o_)}
                if io_:
                    secondary[f"gemm{n}_{p_}"]["operands"] = "bf16 in HBM (A MN-major and B K-major, read in place)"
                del ga_, gb_
            del ga, gb, gc
        n = 1024
        ga = torch.rand(n * n, device=dev) * 2 - 1
        gb = torch.rand(n * n, device=dev) * 2 - 1
        gc = torch.empty(n * n, device=dev)
        gshape = tk.GemmShape(n, n, n)
        for p_ in ("fp32", "tf32", "bf16"):
            cfg = None  # library tile (exact: sized to fill the SMs)
            for _ in range(3):
                tk.gemm_dev(gb, ga, None, gc, gshape, cfg, precision=p_, stream=stream)
            ts = []
            for _ in range(20):
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                tk.gemm_dev(gb, ga, None, gc, gshape, cfg, precision=p_, stream=stream)
                b_.record(stream)
                b_.synchronize()
                ts.append(a_.elapsed_time(b_))
            ms = float(np.median(ts))
            # Device time without host work: 20 calls captured in a graph.
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(stream)
            gg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gg, stream=cap):
                for _ in range(20):
                    tk.gemm_dev(gb, ga, None, gc, gshape, cfg, precision=p_, stream=cap)
            gg.replay()
            torch.cuda.synchronize()
            reps_ = []
            for _ in range(5):  # median of 5 replays (a single one swings with the clock)
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                gg.replay()
                b_.record(stream)
                b_.synchronize()
                reps_.append(a_.elapsed_time(b_) / 20)
            dms = float(np.median(reps_))
            del gg
            pk = {"fp32": 148 * 128 * 1.965e9 / 1e12, "tf32": peaks["bf16_tflops"] / 2.0,
                  "bf16": peaks["bf16_tflops"]}[p_]
            secondary[f"sgemm1024_{p_}"] = {
                "value": round(2 * n ** 3 / (dms * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
                "ms": round(dms, 4), "frac_of_peak": round(2 * n ** 3 / (dms * 1e-3) / 1e12 / pk, 4),
                "api_ms": round(ms, 4),
                "api_gflops": round(2 * n ** 3 / (ms * 1e-3) / 1e9, 1),
                "plan": gemm_plan_str(tk, gshape, tk.exec_options(p_)),
                "note": "value/ms: device time (graph of 20 calls, median of 5 replays); api_*: one tk_gemm_dev call "
                        "between events (host work included); L2-resident operands (12.6 MB); "
                        "fp32 peak = FMUL+FADD issue cap 37.2 TF/s"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ref = CpuReference()
        ref.full_pass()  # warm caches / thread pools
        fl, sec = ref.full_pass()
        cpu = {"value": round(fl / sec / 1e9, 3), "unit": "GFLOP/s", "cores": ref.cores,
               "kind": ref.kind,
               "sample": "one full VGG16 conv stack at batch 1 (1/32 of a GPU step), reference "
                         "conv2d with its fastest CPU algorithm per layer",
               "seconds": round(sec, 3)}

    if rank == 0:
        line = {
            "metric": "VGG16 conv-stack GFLOP/s (conv_flops / time)",
            "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"tf32": "tf32", "bf16": "bf16", "fp32": "f32"}[prec],
            "data": "synthetic (uniform[-1,1) via torch, per-layer independent inputs)",
            "config": {"workload": "VGG16 13 conv layers (3x3/s1/Same, NHWC fp32)",
                       "batch_per_gpu": N, "global_batch": N * world,
                       "algorithm": "im2col implicit GEMM",
                       "precision": prec, "step_gflop": round(step_flops / 1e9, 2),
                       "l2": "flushed between steps (256 MiB write, outside events)",
                       "pre_step": (f"GPU spin of {prespin} cycles before the start event (the step graph "
                                    "is queued before the GPU reaches it)") if prespin else None,
                       "tuning_db": ([os.path.relpath(p_, ROOT) for p_ in db_paths] if db_records else None),
                       "tuning_db_entries": db_records},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": dict(clocks.summary(), samples_in_timed=timed_samples,
                           samples_after_timed=len(clocks.lines) - timed_samples),
            "step_ms": {"min": round(float(np.min(times)), 4),
                        "median": round(float(np.median(times)), 4),
                        "max": round(float(np.max(times)), 4)},
            "layers": layer_rows,
            "multi_gpu": multi,
            "secondary": secondary,
        }
        # Compact digest LAST in the line (a log tail shows it whole).
        summ = {"vgg16_" + prec + "_gflops": round(value, 1), "e2e_gflops": e2e and e2e["value"],
                "roofline_frac": roofline["frac"]}
        for key in ("vgg16_tf32", "vgg16_bf16", "vgg16_bf16_io", "vgg16_3xtf32", "vgg16_fp32",
                    "resnet50_tf32", "resnet50_bf16", "resnet50_bf16_io", "resnet50_tiled_fp32", "sgemm1024_fp32", "sgemm1024_tf32",
                    "sgemm1024_bf16", "gemm4096_tf32", "gemm4096_bf16", "gemm4096_bf16_io",
                    "gemm8192_tf32", "gemm8192_bf16", "gemm8192_bf16_io"):
            if key in secondary:
                v = secondary[key]
                summ[key] = {"gflops": v["value"], "ms": v.get("ms_per_step", v.get("ms"))}
        if "gemm8192_tf32_panels" in multi:
            summ["gemm8192_tf32_panels_gflops"] = multi["gemm8192_tf32_panels"]["value"]
        if "verify" in multi:
            summ["shards_verified"] = multi["verify"]["shards_bitwise_equal_to_recompute"]
        line["summary"] = summ
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
