"""CPU: the C-ABI library loads, exports exactly what include/tk_b200.h
declares, enforces the reference's budgets/grammars host-side, and refuses
to compute without a B200 (there is no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tk_b200.h")).read()
    return sorted(set(re.findall(r"TK_API\s+[\w\s\*]+?\b(tk_\w+)\s*\(", text)))


def test_header_and_exports_agree(tk):
    declared = header_symbols()
    assert declared == sorted(tk.EXPORTS)
    lib = tk.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.tk_abi_version() == 1


def test_no_cpu_fallback(tk):
    if tk.device_count() > 0:
        pytest.skip("a GPU is present")
    shape = tk.ConvShape(1, 5, 5, 4, 4, 3, 3)
    x = np.zeros(shape.in_shape, np.float32)
    w = np.zeros(shape.filt_shape, np.float32)
    with pytest.raises(tk.DeviceError, match="no CPU"):
        tk.conv2d(x, w, shape, tk.parse_conv_params("naive"))
    g = tk.GemmShape(4, 4, 4)
    with pytest.raises(tk.DeviceError):
        tk.gemm_tiled(np.zeros(16), np.zeros(16), None, g, tk.parse_gemm_config("4x4_8x8_loc"),
                      tk.b200_device())


def test_validate_config_matches_reference_verdicts(tk):
    gpu = tk.find_device("Intel Core i7-6700K GPU")
    ok, msg = tk.validate_config(tk.parse_gemm_config("4x4_8x8_loc"), gpu)
    assert ok and msg == "valid"
    # test_gemm.cpp:188-195: three simultaneous violations
    tiny = tk.DeviceSpec("tiny", 64, 1024, 1, 20, 16)
    ok, msg = tk.validate_config(tk.parse_gemm_config("8x4_16x16_loc"), tiny)
    assert not ok and len(msg.split("; ")) == 3
    ok, msg = tk.validate_config(tk.parse_gemm_config("4x4_8x8_loc"), tk.find_device("mali"))
    assert not ok and "local-memory budget" in msg


def test_gemm_tiled_rejects_before_touching_the_gpu(tk):
    g = tk.GemmShape(8, 8, 8)
    z = np.zeros(64, np.float32)
    with pytest.raises(tk.ConfigError, match="local-memory budget"):
        tk.gemm_tiled(z, z, z, g, tk.parse_gemm_config("4x4_8x8_loc"), tk.find_device("mali"))
    cfg = tk.parse_gemm_config("4x4_8x8_noloc")
    cfg.k_step = 0
    with pytest.raises(tk.ConfigError, match="k_step"):
        tk.gemm_tiled(z, z, z, g, cfg, tk.find_device("mali"))


def test_conv_capability_errors(tk):
    x = np.zeros((1, 8, 8, 4), np.float32)
    w = np.zeros((3, 3, 4, 2), np.float32)
    s3 = tk.ConvShape(1, 8, 8, 4, 2, 3, 3, 3, True)
    with pytest.raises(tk.CapabilityError, match="stride 3"):
        tk.conv2d(x, w, s3, tk.parse_conv_params("tiled_t2x2_v4x4"))
    s2 = tk.ConvShape(1, 8, 8, 4, 2, 3, 3, 2, True)
    with pytest.raises(tk.CapabilityError, match="stride 2"):
        tk.conv2d(x, w, s2, tk.parse_conv_params("winograd_t2x2"))
    s1 = tk.ConvShape(1, 8, 8, 4, 2, 3, 3, 1, True)
    with pytest.raises(tk.CapabilityError, match="3x3 output tile"):
        tk.conv2d(x, w, s1, tk.parse_conv_params("winograd_t3x3"))
    bad = tk.ConvShape(1, 2, 2, 4, 2, 3, 3, 1, False)
    with pytest.raises(tk.ShapeError, match="does not fit"):
        tk.conv2d(np.zeros((1, 2, 2, 4), np.float32), w, bad, tk.parse_conv_params("naive"))


def test_grammars(tk):
    for name in ["4x4_8x8_loc", "8x4_8x16_loc_db", "8x2_4x16_noloc"]:
        assert tk.parse_gemm_config(name).name() == name
    for bad in ["4x4_8x8", "4x4_8x8_noloc_db", "0x4_8x8_loc", "4X4_8x8_loc"]:
        with pytest.raises(tk.ParseError):
            tk.parse_gemm_config(bad)
    for name in ["naive", "im2col", "tiled_t4x5_v4x2", "winograd_t2x2"]:
        assert tk.parse_conv_params(name).name() == name
    with pytest.raises(tk.ParseError):
        tk.parse_conv_params("tiled_t4x5_v3x2")


def test_b200_device_spec(tk):
    d = tk.b200_device()
    assert d.cache_line_bytes == 128 and d.register_budget == 255
    assert d.local_memory_bytes >= 227 * 1024 and d.max_workgroup_size == 1024
    assert d.compute_units in (148, 132, 160) or d.compute_units > 0
    ok, _ = tk.validate_config(tk.parse_gemm_config("8x8_16x16_loc_db"), d)
    assert ok


def test_undersized_operands_raise_shape_error(tk):
    """the Python wrappers check buffer sizes before any pointer
    reaches the C ABI (reference check_gemm_operands / check_conv_operands,
    gemm.hpp:165-186, conv.hpp:30-66)."""
    g = tk.GemmShape(8, 8, 8)
    cfg = tk.parse_gemm_config("4x4_8x8_noloc")
    dev = tk.find_device("mali")
    z, small = np.zeros(64, np.float32), np.zeros(63, np.float32)
    with pytest.raises(tk.ShapeError, match="operand A"):
        tk.gemm_tiled(small, z, z, g, cfg, dev)
    with pytest.raises(tk.ShapeError, match="operand B"):
        tk.gemm_naive(z, small, z, g)
    with pytest.raises(tk.ShapeError, match="operand C"):
        tk.gemm_naive(z, z, small, g)
    with pytest.raises(tk.ShapeError, match="operand A"):
        tk.gemm_batched_strided(small, z, 1, 8, 8, 8)
    s = tk.ConvShape(1, 8, 8, 4, 2, 3, 3)
    x = np.zeros(s.in_shape, np.float32)
    w = np.zeros(s.filt_shape, np.float32)
    with pytest.raises(tk.ShapeError, match="input"):
        tk.conv2d(x[:, :7], w, s, tk.parse_conv_params("naive"))
    with pytest.raises(tk.ShapeError, match="filter"):
        tk.conv2d(x, w[..., :1], s, tk.parse_conv_params("im2col"))
    with pytest.raises(tk.ShapeError, match="input"):
        tk.im2col(x[:, :, :7], s)
    import torch
    with pytest.raises(tk.ContractError, match="CUDA tensor"):
        tk.conv2d_dev(torch.zeros(s.in_shape), torch.zeros(s.filt_shape),
                      torch.zeros(s.out_shape), s, tk.parse_conv_params("im2col"))
    with pytest.raises(tk.ContractError, match="CUDA tensor"):
        tk.gemm_dev(torch.zeros(64), torch.zeros(64), None, torch.zeros(64), g)


def test_tuning_db_drives_the_plan(tk, tmp_path):
    """lookup_best on the launch path: with a DB loaded, a call whose
    tensor-core knobs are automatic takes the fastest valid record's knobs
    for its (problem, algorithm, precision); explicit knobs still win, and
    clearing the DB restores the built-in rules.  Host-side (plan only)."""
    s = tk.ConvShape(32, 56, 56, 256, 256, 3, 3, 1, True)
    im = tk.parse_conv_params("im2col")
    base = tk.conv2d_plan_info(s, im, "tf32")
    assert base["kernel"] == "tc_im2col" and base["tuned"] == 0
    key = s.key()
    db = tmp_path / "db.ndjson"
    recs = [
        {"problem": key, "config": "im2col@tf32", "median_ns": 170000, "valid": True},
        {"problem": key, "config": "im2col@tf32_c2_pixn", "median_ns": 150000, "valid": True},
        {"problem": key, "config": "im2col@tf32_halo", "median_ns": 100000, "valid": False},
        {"problem": key, "config": "im2col@bf16_halo", "median_ns": 90000, "valid": True},
        {"problem": key, "config": "tiled_t2x2_v4x8", "median_ns": 5000000, "valid": True},
    ]
    import json
    db.write_text("\n".join(json.dumps(dict(r, device="NVIDIA B200", samples=5, min_ns=1,
                                             mean_ns=1, gflops=1.0)) for r in recs) + "\n")
    try:
        assert tk.tuning_db_load(str(db)) >= 2
        d = tk.conv2d_plan_info(s, im, "tf32")
        assert d["tuned"] == 1 and d["kernel"] == "tc_pixn" and d["cta_group"] == 2
        assert tk.conv2d_plan_info(s, im, "bf16")["kernel"] == "tc_halo"
        # explicit knobs are the caller's
        d = tk.conv2d_plan_info(s, im, options=tk.exec_options("tf32", mode="im2col"))
        assert d["tuned"] == 0 and d["kernel"] == "tc_im2col"
        # other shapes keep the rules
        s2 = tk.ConvShape(32, 28, 28, 512, 512, 3, 3, 1, True)
        assert tk.conv2d_plan_info(s2, im, "tf32")["tuned"] == 0
    finally:
        tk.tuning_db_clear()
    assert tk.tuning_db_size() == 0
    assert tk.conv2d_plan_info(s, im, "tf32")["kernel"] == "tc_im2col"
    with pytest.raises(tk.IoError):
        tk.tuning_db_load(str(tmp_path / "missing.ndjson"))


def test_gemm_plan_info_host_only(tk):
    """tk_gemm_plan_info (what tk_gemm_dev would run) is host logic: it
    answers without a GPU, follows the cost model, the knobs and the DB."""
    d = tk.gemm_plan_info(tk.GemmShape(1024, 1024, 1024), precision="fp32")
    assert d["kernel"] == "exact_simt" and d["precision"] == "fp32" and d["splits"] == 1
    d = tk.gemm_plan_info(tk.GemmShape(1024, 1024, 1024), precision="tf32")
    assert d["kernel"] == "tc_plain" and d["tile_m"] == 128 * d["cta_group"]
    assert d["a_in_place"] and d["b_in_place"]  # nn: A MN-major, B K-major, read where they lie
    d = tk.gemm_plan_info(tk.GemmShape(1024, 1024, 1024), precision="3xtf32")
    assert d["k_depth"] == 3 * 1024 and not d["a_in_place"]
    d = tk.gemm_plan_info(tk.GemmShape(512, 512, 512),
                          options=tk.exec_options("tf32", tile_n=128, cluster=1, split=1))
    assert (d["cta_group"], d["tile_n"], d["splits"]) == (1, 128, 1)
    with pytest.raises(tk.ShapeError):
        tk.gemm_plan_info(tk.GemmShape(0, 4, 4), precision="tf32")


def test_committed_tuning_dbs_load_and_steer_plans(tk):
    """The DBs bench.py loads parse (the reference's NDJSON schema + the B200
    keys), and the plan queries report their choices -- host logic, no GPU."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    conv_db = os.path.join(root, "profiles", "r02_tune_ncu.ndjson")
    gemm_db = os.path.join(root, "profiles", "r02_tune_gemm.ndjson")
    tk.tuning_db_clear()
    try:
        assert tk.tuning_db_load(conv_db) > 0 and tk.tuning_db_load(gemm_db) > 0
        # a tuned GEMM record steers the GEMM plan
        rec = next(json.loads(ln) for ln in open(gemm_db)
                   if "_" in json.loads(ln)["config"].split("@")[1])
        m, n, k = (int(v) for v in re.match(r"gemm_nn_m(\d+)_n(\d+)_k(\d+)", rec["problem"]).groups())
        assert tk.gemm_plan_info(tk.GemmShape(m, n, k), precision=rec["precision"])["tuned"] == 1
        # a tuned conv record (fp32 activations) steers the conv plan
        for ln in open(conv_db):
            r = json.loads(ln)
            fam, rest = r["config"].split("@")
            if fam == "im2col" and "_" in rest and r["problem"].startswith("conv_n32_"):
                g = re.match(r"conv_n(\d+)_(\d+)x(\d+)x(\d+)_k(\d+)_f(\d+)x(\d+)_s(\d+)_", r["problem"])
                nb, h, w, c, kk, fr, fc, st = (int(v) for v in g.groups())
                shape = tk.ConvShape(nb, h, w, c, kk, fr, fc, st, True)
                assert tk.conv2d_plan_info(shape, tk.parse_conv_params("im2col"),
                                           r["precision"])["tuned"] == 1, r["config"]
                break
        else:
            pytest.fail("no tuned conv record")
    finally:
        tk.tuning_db_clear()
