"""The reference's C++ API recompiled unchanged against include/tilekit and
linked to libtilekit_b200.so (the drop-in boundary).  The CPU run covers the
host logic (grammars, budgets, geometry, error classes); the GPU run covers
the arithmetic."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1904_05347_b200")
INC = os.path.join(ROOT, "include", "tilekit")


def build(name):
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    exe = os.path.join(ROOT, "tests", "cpp", name)
    newest = max([os.path.getmtime(src)] +
                 [os.path.getmtime(os.path.join(INC, f)) for f in os.listdir(INC)])
    if not os.path.exists(exe) or os.path.getmtime(exe) < newest:
        subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                        src, "-o", exe, "-L", LIBDIR, "-ltilekit_b200",
                        f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


ARGS = [os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "data")]
NAMES = ["test_dropin", "test_tuner", "test_analysis"]


@pytest.mark.parametrize("name", NAMES)
def test_cpp_host_logic(name, tmp_path):
    r = subprocess.run([build(name), "cpu"] + ARGS, capture_output=True, text=True, timeout=120,
                       cwd=tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_cpp_gpu(name, tmp_path):
    r = subprocess.run([build(name), "gpu"] + ARGS, capture_output=True, text=True, timeout=900,
                       cwd=tmp_path)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
