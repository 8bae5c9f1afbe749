"""The checked build (libtilekit_b200_checked.so: TKB_DCHECK device-side
invariants of the hand-written indexing on -- shared-memory layout,
staging / TMEM / tail / split slots, narrow-halo tap tables, gather and pad
source ranges, exact-path output offsets).  compute-sanitizer is closed on
this GPU pool; this is its stand-in: one launch of every kernel mode
(tools/sanitize_cases.py, each also checked against the oracle) plus every
bench layer shape at batch 32 in TF32 / BF16 / BF16 with bf16 activations,
all under the checks.  A violated invariant traps the launch and fails the
run with the failing site printed."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1904_05347_b200", "libtilekit_b200_checked.so")


def test_checked_library_exports_the_abi():  # CPU: loads, no launches
    import ctypes
    if not os.path.exists(CHECKED):
        pytest.skip("checked build not built (make -C paper_1904_05347_b200 checked)")
    lib = ctypes.CDLL(CHECKED)
    for sym in ("tk_gemm_dev", "tk_conv2d_dev", "tk_conv2d_plan_info", "tk_tuning_db_load"):
        assert hasattr(lib, sym), sym


@pytest.mark.gpu
@pytest.mark.timeout(1200)
def test_every_mode_under_device_checks():
    assert os.path.exists(CHECKED), "checked build missing: __graft_entry__.build() makes it"
    env = dict(os.environ, TK_LIB_PATH=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), "--bench"],
                       env=env, capture_output=True, text=True, timeout=1100, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "all ok" in r.stdout, out[-4000:]
    assert "TKB_DCHECK failed" not in out


@pytest.mark.gpu
@pytest.mark.timeout(1200)
@pytest.mark.parametrize("lib", ["release", "checked"])
def test_forced_stream_k_tail(lib):
    """The stream-K tail (balanced last wave: partial pieces + ordered
    reduction) is rarely chosen by the cost model on the bench shapes, so
    run every kernel mode and every bench layer with it forced
    (TK_EXPERIMENTS=1 TK_TAIL_FORCE=1): oracle parity per mode, finite
    outputs per bench layer, and -- with the checked build -- the slot
    invariants."""
    env = dict(os.environ, TK_EXPERIMENTS="1", TK_TAIL_FORCE="1")
    if lib == "checked":
        assert os.path.exists(CHECKED), "checked build missing: __graft_entry__.build() makes it"
        env["TK_LIB_PATH"] = CHECKED
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), "--bench"],
                       env=env, capture_output=True, text=True, timeout=1100, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "all ok" in r.stdout, out[-4000:]
