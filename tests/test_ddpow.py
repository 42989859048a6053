"""Host check of the certified double-double pow (csrc/ddpow.cuh) behind the
device weight synthesiser: compiled for the host (the header is
__host__ __device__), every result it certifies equals glibc pow — the function
weights.cpp:118-122 calls — over the inverse-CDF arguments of the C1, C3, C4
and C5 recipes; about 1/16 of the draws are left to the host's libm."""
import os
import re
import subprocess

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_ddpow.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_ddpow")


def test_certified_pow_equals_glibc():
    flags = ["-mfma"] if "fma" in open("/proc/cpuinfo").read() else []
    subprocess.run(["g++", "-O2", "-std=c++17", *flags, "-ffp-contract=off", "-x", "c++", SRC, "-o", BIN],
                   check=True, capture_output=True, text=True)
    out = subprocess.run([BIN, "400000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    m = re.search(r"total (\d+) flagged (\d+) .* mismatches (\d+)", out.stdout)
    assert m and int(m.group(3)) == 0
    assert 0.05 < int(m.group(2)) / int(m.group(1)) < 0.075
