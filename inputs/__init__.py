"""The five BASELINE.json workloads (C1-C5) as seeded synthetic weight arrays.

Input preparation shared by BOTH bench arms and the tests; it is neither the
product (``paper_1406_1215_b200``, ``libclgen_b200.so``) nor the checker
(``oracle/``), so the reference arm (``bench.py --impl reference``) never maps
the product library or touches the GPU.

Recipes follow SURVEY.md §8(d).  Weights are synthesised ONCE on the host by
the reference's own synthesiser arithmetic (``libclgen_inputs.so``: the
sequential xoshiro synth stream + glibc pow, bit-identical to
weights.cpp:103-128; tested against the reference's ``synth_powerlaw`` in
tests/test_oracle.py), then sorted descending on the host with all cores
(values only; the stable label order of make_weight_sequence does not change
them).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libclgen_inputs.so")
_L = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """g++ -O2 (no -march: x86-64 SSE2, no FMA, glibc libm, as the reference build)."""
    src = os.path.join(HERE, "synth.cpp")
    hdr = os.path.join(HERE, "clgen_inputs.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return LIB_PATH
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-shared", "-pthread",
                    "-o", LIB_PATH, src], check=True)
    return LIB_PATH


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    desc: str
    seed: int = 7           # generation seed
    materialise: bool = False


WORKLOADS = {
    "c1": Workload("c1", 1_000_000,
                   "discrete PL gamma=2.5 on [10,1000], materialised uint32 pairs", materialise=True),
    "c2": Workload("c2", 10_000_000, "uniform w=50 (Erdos-Renyi limit), materialised", materialise=True),
    "c3": Workload("c3", 100_000_000, "PL gamma=2.1 on [2,1e5], streaming fold"),
    "c4": Workload("c4", 1_000_000_000, "PL gamma=2.5 scaled to mean 500, streaming fold"),
    "c5": Workload("c5", 10_000_000, "saturated core gamma=2.0, w_max=sqrt(S), streaming fold"),
}


def _host():
    global _L
    with _lock:
        if _L is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = C.CDLL(LIB_PATH)
            _declare(L)
            _L = L
    return _L


def _declare(L):
    L.clgen_host_powerlaw_draws.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double,
                                            C.c_uint64, C.c_void_p, C.c_int]
    L.clgen_host_discrete_powerlaw.argtypes = [C.c_int64, C.c_double, C.c_int64, C.c_int64,
                                               C.c_uint64, C.c_void_p, C.c_int]
    L.clgen_host_sort_desc.argtypes = [C.c_void_p, C.c_int64, C.c_int]


def _threads() -> int:
    return os.cpu_count() or 1


class InputError(ValueError):
    """The reference synthesiser's contract violations (weights.cpp:105-108)."""


def sort_desc(w: np.ndarray) -> np.ndarray:
    """In-place parallel descending sort of the values on the host."""
    if _host().clgen_host_sort_desc(w.ctypes.data, w.size, _threads()) != 0:
        raise InputError("sort_desc: bad arguments")
    return w


def powerlaw(n: int, gamma: float, w_min: float, w_max: float, seed: int,
             sort: bool = True) -> np.ndarray:
    """synth_powerlaw(n, gamma, w_min, w_max, seed).weights (weights.cpp:103-128)."""
    out = np.empty(n, np.float64)
    if _host().clgen_host_powerlaw_draws(n, gamma, w_min, w_max, seed, out.ctypes.data,
                                         _threads()) != 0:
        raise InputError("synth_powerlaw: bad arguments")
    return sort_desc(out) if sort else out


def discrete_powerlaw(n: int, gamma: float, k_min: int, k_max: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    if _host().clgen_host_discrete_powerlaw(n, gamma, k_min, k_max, seed, out.ctypes.data,
                                            _threads()) != 0:
        raise InputError("discrete_powerlaw: bad arguments")
    return sort_desc(out)


def _blocked_sum_host(w: np.ndarray) -> float:
    """weights.cpp:21-30 on the host (input preparation only): the column-wise
    left fold over a [blocks, 4096] view is each block's sequential fold."""
    n = w.size
    nf = n // 4096
    parts = []
    if nf:
        blocks = w[: nf * 4096].reshape(nf, 4096)
        acc = np.zeros(nf)
        for k in range(4096):
            acc += blocks[:, k]
        parts = acc.tolist()
    if n % 4096:
        t = 0.0
        for x in w[nf * 4096:].tolist():
            t += x
        parts.append(t)
    total = 0.0
    for x in parts:
        total += x
    return total


def make(name: str, n: int | None = None) -> np.ndarray:
    """Weights of workload `name` (c1..c5), optionally at a reduced n."""
    wl = WORKLOADS[name]
    n = n or wl.n
    if name == "c1":
        return discrete_powerlaw(n, 2.5, 10, 1000, 1)
    if name == "c2":
        return np.full(n, 50.0)
    if name == "c3":
        return powerlaw(n, 2.1, 2.0, 1e5, 1)
    if name == "c4":
        # synth_powerlaw(n, 2.5, 1, 1000, seed=1) x (500 / mean)
        w = powerlaw(n, 2.5, 1.0, 1000.0, 1)
        mean = _blocked_sum_host(w) / n
        w *= 500.0 / mean
        return w
    if name == "c5":
        return saturated_core(n)
    raise KeyError(name)


def saturated_core(n: int, gamma: float = 2.0, stretch: float = 1.047, seed: int = 1,
                   iters: int = 8) -> np.ndarray:
    """C5: continuous PL on [1, stretch*c] clamped at c, iterated to c = sqrt(S),
    then c bumped by ulps until c*c/S >= 1 (the top core hits p = 1)."""
    draws = None
    c = math.sqrt(n * 10.0)
    for _ in range(iters):
        draws = powerlaw(n, gamma, 1.0, stretch * c, seed, sort=False)
        np.minimum(draws, c, out=draws)
        S = float(draws.sum())
        c_new = math.sqrt(S)
        if abs(c_new - c) <= 1e-9 * c:
            c = c_new
            break
        c = c_new
    w = sort_desc(np.minimum(powerlaw(n, gamma, 1.0, stretch * c, seed, sort=False), c))
    S = _blocked_sum_host(w)
    core = w == w[0]
    while c * c / S < 1.0:
        c = math.nextafter(c, math.inf)
        w[core] = c  # raise the clamped core to the bumped cap
        S = _blocked_sum_host(w)
    return w
