"""The reference's C++ API recompiled unchanged against include/tilekit and
linked to libtilekit_b200.so (the drop-in boundary).  The CPU run covers the
host logic (grammars, budgets, geometry, error classes); the GPU run covers
the arithmetic."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1904_05347_b200")
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build():
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(src):
        subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                        src, "-o", BIN, "-L", LIBDIR, "-ltilekit_b200",
                        f"-Wl,-rpath,{LIBDIR}"], check=True)
    return BIN


def test_dropin_compiles_and_host_logic():
    r = subprocess.run([build(), "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_gpu():
    r = subprocess.run([build(), "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
