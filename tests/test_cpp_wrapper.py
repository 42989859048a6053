"""The header-only C++ mirror (include/clgen_b200.hpp) compiles against the
C ABI here (CPU) and passes the reference-style checks on a GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_wrapper.cpp")
PKG = os.path.join(ROOT, "paper_1406_1215_b200")
BIN = os.path.join(ROOT, "tests", "cpp", "test_wrapper")


def build():
    from paper_1406_1215_b200 import build as b
    b.build()
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
           "-L", PKG, "-lclgen_b200", f"-Wl,-rpath,{PKG}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


def test_wrapper_compiles():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_wrapper_runs_on_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([build()], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout
