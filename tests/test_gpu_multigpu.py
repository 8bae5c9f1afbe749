"""Multi-GPU path of bench.py: the library runs on every
rank (no oracle), each rank owns a batch slice of one logical tensor / a
column panel of one GEMM, and the shards gathered to rank 0 over NCCL match
rank 0's own recomputation bit for bit.  The 2-rank case needs two GPUs
(skipped on a 1-GPU box); the 1-rank case exercises the same code on one."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def run_bench(gpus):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--steps", "3",
           "--warmup", "3", "--no-secondary", "--no-cpu", "--no-e2e", "--no-layers"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert lines, out.stdout[-2000:] + out.stderr[-2000:]
    return json.loads(lines[-1])


@pytest.mark.timeout(900)
@pytest.mark.parametrize("gpus", [1, 2])
def test_sharded_stack_and_gemm_panels(gpus):
    import torch
    if torch.cuda.device_count() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    d = run_bench(gpus)
    assert d["n_gpus"] == gpus
    m = d["multi_gpu"]
    assert m["ranks"] == gpus and len(m["rank_ms_per_step"]) == gpus
    assert m["global_batch"] == 32 * gpus
    assert m["verify"]["shards_bitwise_equal_to_recompute"] is True
    assert m["verify"]["max_scaled_error_vs_fp32_exact_img0"] <= 1e-3
    g = m["gemm8192_tf32_panels"]
    assert g["verify_first_256_cols_bitwise"] is True
    assert len(g["rank_ms"]) == gpus and g["panel_cols"] == 8192 // gpus
