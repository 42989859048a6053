"""CPU tests of the drop-in boundary: the sm_100a library loads without a GPU
and exports exactly the C-ABI entry points include/clgen_dev.h declares."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "clgen_dev.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(clgen_(?:dev|spmd)_\w+)\s*\(", src, re.M)))


def lib_path():
    from paper_1406_1215_b200 import build
    return build.build()


def test_header_declares_entry_points():
    names = declared()
    assert "clgen_dev_create_edges_range" in names
    assert "clgen_dev_stream_range" in names
    assert "clgen_spmd_generate" in names
    assert len(names) >= 10


def test_library_exports_every_declared_symbol():
    path = lib_path()
    lib = ctypes.CDLL(path)
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(clgen_(?:dev|spmd)_\w+)\b", out))
    assert set(declared()) <= exported


def test_python_binding_lists_every_symbol():
    from paper_1406_1215_b200 import _lib
    assert set(_lib.EXPORTS) == set(declared())


def test_sm100a_code_in_library():
    path = lib_path()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1406_1215_b200 import api, error
    with pytest.raises(error):
        api.Device(0)
