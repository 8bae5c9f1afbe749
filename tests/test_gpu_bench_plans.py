"""GPU parity at exactly the configurations bench.py times.

Every distinct VGG-16 (9) and ResNet-50 (21) conv shape at batch 32 -- the
per-GPU shard of BASELINE configs[4], the plans the headline and the
secondary stacks run (tail plan, split-K count, flat rows, multi-image
tiles, halo width, resident filter all depend on N) -- through the bench's
own call sequence: tk_conv2d_workspace_size, tk_conv2d_prepare_dev,
tk_conv2d_run_dev.  Images {0, 15, 31} are checked against single-image runs
of the oracle (conv2d_naive, reference conv.hpp:74-113; batch independence,
test_conv.cpp:268-293), in every precision:

  fp32    bit-identical (max_rel_error == 0)
  tf32    max_scaled_error <= 1e-3
  bf16    max_scaled_error <= 5e-3 (the EFFECTIVE precision from
          tk_conv2d_plan_info decides the bar: a BF16 request that runs in
          TF32 is reported and held to the TF32 bar)
  3xtf32  max_scaled_error <= 5e-5

The oracle result of a (layer, image) is computed once and shared by the
four precisions.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import RESNET50, VGG16  # noqa: E402

N = 32
IMAGES = (0, 15, 31)
TOL = {"tf32": 1e-3, "bf16": 5e-3, "3xtf32": 5e-5}

LAYERS = [(name, 3, 1, h, c, k) for name, h, c, k, _ in VGG16] + \
         [(name, r, s, h, c, k) for name, r, s, h, c, k, _ in RESNET50]

_inputs = {}
_want = {}


def _host_inputs(tk, idx):
    """Selected images of the layer's seeded batch-32 input + its filter."""
    import torch
    name, r, s, h, c, k = LAYERS[idx]
    if idx not in _inputs:
        gen = torch.Generator(device="cuda").manual_seed(1000 + idx)
        x = torch.rand((N, h, h, c), device="cuda", generator=gen) * 2 - 1
        f = torch.rand((r, r, c, k), device="cuda", generator=gen) * 2 - 1
        _inputs[idx] = ({i: x[i:i + 1].cpu().numpy() for i in IMAGES}, f.cpu().numpy())
        del x, f
    return _inputs[idx]


def _device_inputs(idx):
    import torch
    name, r, s, h, c, k = LAYERS[idx]
    gen = torch.Generator(device="cuda").manual_seed(1000 + idx)
    x = torch.rand((N, h, h, c), device="cuda", generator=gen) * 2 - 1
    f = torch.rand((r, r, c, k), device="cuda", generator=gen) * 2 - 1
    return x, f


def _oracle(oracle, tk, idx, img):
    key = (idx, img)
    if key not in _want:
        name, r, s, h, c, k = LAYERS[idx]
        xs, f = _host_inputs(tk, idx)
        conv = oracle.Conv(1, h, h, c, k, r, r, s, True)
        _want[key] = oracle.conv2d_naive(conv, xs[img], f)
    return _want[key]


def _run(tk, idx, prec, x, f):
    import torch
    name, r, s, h, c, k = LAYERS[idx]
    shape = tk.ConvShape(N, h, h, c, k, r, r, s, True)
    algo = tk.parse_conv_params("im2col")
    ws = torch.empty(max(tk.conv2d_workspace_size(shape, algo, prec), 4) // 4 + 1, device="cuda")
    y = torch.full(shape.out_shape, float("nan"), device="cuda")
    side = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    side.wait_stream(main)
    # the bench forks the filter prepare to a side stream and joins before run
    tk.conv2d_prepare_dev(f, shape, algo, ws, precision=prec, stream=side)
    main.wait_stream(side)
    tk.conv2d_run_dev(x, f, y, shape, algo, ws, precision=prec, stream=main)
    torch.cuda.synchronize()
    return y


DB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                  "r02_tune_ncu.ndjson")


@pytest.fixture(params=["rules", "tuned"])
def knob_source(request, tk):
    """The plans of the built-in rules, and those of the committed tuning DB
    that bench.py loads (tk_tuning_db_load)."""
    tk.tuning_db_clear()
    if request.param == "tuned":
        if not os.path.exists(DB):
            pytest.skip("no tuning DB")
        tk.tuning_db_load(DB)
    yield request.param
    tk.tuning_db_clear()


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("prec", ["tf32", "bf16", "3xtf32", "fp32"])
@pytest.mark.parametrize("idx", range(len(LAYERS)), ids=[lay[0] for lay in LAYERS])
def test_bench_layer_batch32(tk, oracle, idx, prec, knob_source):
    name, r, s, h, c, k = LAYERS[idx]
    shape = tk.ConvShape(N, h, h, c, k, r, r, s, True)
    plan = tk.conv2d_plan_info(shape, tk.parse_conv_params("im2col"), prec)
    assert plan["requested_precision"] == prec
    if knob_source == "tuned" and not plan["tuned"]:
        pytest.skip("the DB keeps the rules' plan for this shape")
    x, f = _device_inputs(idx)
    y = _run(tk, idx, prec, x, f)
    assert not bool(torch_isnan_any(y)), (name, prec, plan)
    for img in IMAGES:
        want = _oracle(oracle, tk, idx, img)
        got = y[img:img + 1].cpu().numpy()
        if prec == "fp32":
            assert plan["precision"] == "fp32"
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (name, img)
        else:
            bar = TOL[plan["precision"]] if plan["precision"] in TOL else TOL[prec]
            err = oracle.max_scaled_error(got, want)
            assert err <= bar, (name, prec, img, err, plan)
    if prec == "tf32":
        # deterministic run to run (ordered split-K / tail reductions)
        y2 = _run(tk, idx, prec, x, f)
        import torch
        assert torch.equal(y.view(torch.int32), y2.view(torch.int32)), (name, plan)


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
@pytest.mark.parametrize("vi", range(len(VGG16)), ids=[v[0] for v in VGG16])
def test_vgg_batch1_plans(tk, oracle, vi, prec, knob_source):
    """BASELINE configs[1] at batch 1 (bench.py's vgg16_batch1 leg): the
    rules' plans and the tuning DB's batch-1 records (halo for conv3_x,
    im2col with K split 8 for conv5, ...) against the oracle."""
    import torch
    name, h, c, k, _ = VGG16[vi]
    shape = tk.ConvShape(1, h, h, c, k, 3, 3, 1, True)
    algo = tk.parse_conv_params("im2col")
    plan = tk.conv2d_plan_info(shape, algo, prec)
    if knob_source == "tuned" and not plan["tuned"]:
        pytest.skip("the DB keeps the rules' plan for this shape")
    gen = torch.Generator(device="cuda").manual_seed(2000 + vi)
    x = torch.rand((1, h, h, c), device="cuda", generator=gen) * 2 - 1
    f = torch.rand((3, 3, c, k), device="cuda", generator=gen) * 2 - 1
    ws = torch.empty(max(tk.conv2d_workspace_size(shape, algo, prec), 4) // 4 + 1, device="cuda")
    ys = []
    for _ in range(2):
        y = torch.full(shape.out_shape, float("nan"), device="cuda")
        tk.conv2d_prepare_dev(f, shape, algo, ws, precision=prec)
        tk.conv2d_run_dev(x, f, y, shape, algo, ws, precision=prec)
        torch.cuda.synchronize()
        ys.append(y)
    want = oracle.conv2d_naive(oracle.Conv(1, h, h, c, k, 3, 3, 1, True), x.cpu().numpy(),
                               f.cpu().numpy())
    bar = TOL[plan["precision"]] if plan["precision"] in TOL else TOL[prec]
    err = oracle.max_scaled_error(ys[0].cpu().numpy(), want)
    assert err <= bar, (name, prec, err, plan)
    assert torch.equal(ys[0].view(torch.int32), ys[1].view(torch.int32)), (name, plan)


def torch_isnan_any(y):
    import torch
    return torch.isnan(y).any().item()


@pytest.mark.parametrize("idx", range(len(LAYERS)), ids=[lay[0] for lay in LAYERS])
def test_plan_reports_effective_precision(tk, idx):  # host-only: runs on CPU too
    """BF16 requests report the arithmetic that actually runs: bf16 on the
    box / halo / pointwise / im2col paths (the C = 3 first layers included,
    through narrow-pixel im2col), tf32 only on the gather producers (fp32
    operands) -- never silently."""
    name, r, s, h, c, k = LAYERS[idx]
    shape = tk.ConvShape(N, h, h, c, k, r, r, s, True)
    plan = tk.conv2d_plan_info(shape, tk.parse_conv_params("im2col"), "bf16")
    assert plan["kernel"] != "tc_gather", plan  # every bench layer has a BF16 path
    if plan["kernel"] == "tc_gather":
        assert plan["precision"] == "tf32"
    else:
        assert plan["precision"] == "bf16"


# bf16 activations in HBM (tk_exec_options.io): the layer reads a bf16 input
# and/or writes a bf16 output -- a BF16 network's layer-to-layer format, no
# conversion pass.  Checked against the oracle on the bf16-rounded input;
# the bar is the BF16 one plus the output's own rounding (2^-9 of |y|).
TOL_BF16_IO = 5e-3 + 2.0 ** -9
_want_b = {}


def _oracle_bf16_in(oracle, idx, img, xb):
    key = (idx, img)
    if key not in _want_b:
        name, r, s, h, c, k = LAYERS[idx]
        conv = oracle.Conv(1, h, h, c, k, r, r, s, True)
        _, f = _host_inputs(None, idx)
        xi = xb[img:img + 1].float().cpu().numpy()
        _want_b[key] = oracle.conv2d_naive(conv, xi, f)
    return _want_b[key]


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("io", ["bf16", "in_bf16", "out_bf16"])
@pytest.mark.parametrize("idx", range(len(LAYERS)), ids=[lay[0] for lay in LAYERS])
def test_bench_layer_bf16_activations(tk, oracle, idx, io, knob_source):
    import torch
    name, r, s, h, c, k = LAYERS[idx]
    if io != "bf16" and idx % 3:
        pytest.skip("mixed in/out formats on every third layer")
    shape = tk.ConvShape(N, h, h, c, k, r, r, s, True)
    algo = tk.parse_conv_params("im2col")
    opts = tk.exec_options("bf16", io=io)
    if knob_source == "tuned":
        # the DB's bf16-activation records (family im2col_io, bench.py's
        # vgg16_bf16_io / resnet50_bf16_io legs)
        if io != "bf16" or not tk.conv2d_plan_info(shape, algo, options=opts)["tuned"]:
            pytest.skip("the DB keeps the rules' plan for this shape / format")
    x, f = _device_inputs(idx)
    xb = x.to(torch.bfloat16)
    xin = xb if io in ("bf16", "in_bf16") else xb.float()  # same values either way
    ws = torch.empty(max(tk.conv2d_workspace_size(shape, algo, options=opts), 4) // 4 + 1,
                     device="cuda")
    ydt = torch.bfloat16 if io in ("bf16", "out_bf16") else torch.float32
    y = torch.full(shape.out_shape, float("nan"), device="cuda", dtype=ydt)
    tk.conv2d_prepare_dev(f, shape, algo, ws, options=opts)
    tk.conv2d_run_dev(xin, f, y, shape, algo, ws, options=opts)
    torch.cuda.synchronize()
    assert not bool(torch.isnan(y.float()).any()), (name, io)
    for img in IMAGES:
        want = _oracle_bf16_in(oracle, idx, img, xb)
        got = y[img:img + 1].float().cpu().numpy()
        err = oracle.max_scaled_error(got, want)
        assert err <= TOL_BF16_IO, (name, io, img, err)
    # the fp32-activation BF16 run on the same (bf16-exact) values agrees to
    # the output rounding
    if io == "bf16":
        y32 = torch.empty(shape.out_shape, device="cuda")
        tk.conv2d_dev(xb.float(), f, y32, shape, algo, options=tk.exec_options("bf16"))
        torch.cuda.synchronize()
        d = (y.float() - y32).abs().max().item() / y32.abs().max().item()
        assert d <= 2.0 ** -8, (name, d)


def test_bf16_activations_need_bf16_im2col(tk):  # host-only checks: CPU too
    """The io flags are a BF16 tensor-core feature of the device-buffer
    calls: TF32 / FP32 / Winograd requests with them are rejected
    (CapabilityError) before anything runs."""
    shape = tk.ConvShape(1, 8, 8, 64, 64, 3, 3, 1, True)
    for prec, algo in (("tf32", "im2col"), ("fp32", "im2col"), ("bf16", "winograd_t2x2")):
        with pytest.raises(tk.CapabilityError):
            tk.conv2d_workspace_size(shape, tk.parse_conv_params(algo),
                                     options=tk.exec_options(prec, io="bf16"))
    im = tk.parse_conv_params("im2col")
    assert tk.conv2d_workspace_size(shape, im, options=tk.exec_options("bf16", io="bf16")) > 0
    # no conversion copy of the input in the workspace when it arrives in bf16
    assert tk.conv2d_workspace_size(shape, im, options=tk.exec_options("bf16", io="in_bf16")) < \
        tk.conv2d_workspace_size(shape, im, options=tk.exec_options("bf16"))


@pytest.mark.gpu
@pytest.mark.parametrize("io", ["bf16", "in_bf16", "out_bf16"])
@pytest.mark.parametrize("shape", [(2, 20, 20, 3, 32, 3, 1), (2, 14, 14, 64, 96, 3, 1),
                                   (2, 9, 9, 256, 48, 1, 1), (1, 30, 30, 3, 64, 7, 2),
                                   (3, 17, 13, 128, 256, 3, 1), (2, 11, 11, 12, 64, 1, 1),
                                   (2, 10, 10, 20, 64, 3, 1), (2, 12, 12, 8, 128, 1, 2),
                                   (1, 8, 8, 4, 64, 3, 2)])
def test_bf16_output_ragged_features(tk, oracle, shape, io):
    """bf16 activations on ragged channel / feature counts (tiles that are
    not 64-feature multiples, channel rows that are not 16-byte multiples):
    either the exact result (within the BF16 + output-rounding bar) or a
    CapabilityError -- never unwritten or garbage elements."""
    import torch
    N, H, C, K, R, st = shape[0], shape[1], shape[3], shape[4], shape[5], shape[6]
    W = shape[2]
    s = tk.ConvShape(N, H, W, C, K, R, R, st, True)
    conv = oracle.Conv(N, H, W, C, K, R, R, st, True)
    x = oracle.fill_random(int(np.prod(conv.in_shape)), 41).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), 42).reshape(conv.filt_shape)
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    want = oracle.conv2d_naive(conv, xb.float().cpu().numpy(), f)
    opts = tk.exec_options("bf16", io=io)
    ydt = torch.bfloat16 if io in ("bf16", "out_bf16") else torch.float32
    y = torch.full(s.out_shape, float("nan"), device="cuda", dtype=ydt)
    xi = xb if io in ("bf16", "in_bf16") else xb.float()
    try:
        tk.conv2d_dev(xi, torch.from_numpy(f).cuda(), y, s, tk.parse_conv_params("im2col"),
                      options=opts)
        torch.cuda.synchronize()
    except tk.CapabilityError:
        return
    got = y.float().cpu().numpy()
    assert not np.isnan(got).any()
    assert oracle.max_scaled_error(got, want) <= TOL_BF16_IO
