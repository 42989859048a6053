"""TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 Chung–Lu generator.

Two CPU implementations of the reference hot path, loaded through ctypes:

* ``port`` — ``oracle/clgen_oracle.c``: our plain-C restatement of
  ``/root/reference/proj/core`` (rng.hpp, edge_skip.cpp, weights.cpp, cost.cpp,
  partition.cpp), each function citing the reference file:line it follows.
* ``ref``  — ``oracle/_ref/libclgen_ref.so``: the UNMODIFIED reference sources
  compiled by ``oracle/Makefile`` plus our extern "C" shim ``ref_driver.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package, and only as the checker / CPU baseline.  The product
package (``paper_1406_1215_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libclgen_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libclgen_ref.so")
REF_SRC = "/root/reference/proj/core"

_i64 = C.c_int64
_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)


class OracleError(RuntimeError):
    """A contract violation reported by the oracle (clgen::error in the reference)."""


def build(ref: bool = True) -> None:
    """Compile the C restatement and, where /root/reference exists, the reference."""
    targets = ["port"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets, f"-j{os.cpu_count() or 4}"], check=True)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t) if a is not None else None


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------------------- port
class _Port:
    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_node_rng_key.restype = _u64
        L.orc_node_rng_key.argtypes = [_u64, _i64]
        L.orc_stream_open01.argtypes = [_u64, _i64, _i64, _dp]
        L.orc_blocked_sum.restype = C.c_double
        L.orc_blocked_sum.argtypes = [_dp, _i64]
        L.orc_expected_total_edges.restype = C.c_double
        L.orc_expected_total_edges.argtypes = [_dp, _i64, C.c_double]
        L.orc_synth_powerlaw.argtypes = [_i64, C.c_double, C.c_double, C.c_double, _u64, _dp]
        L.orc_skip_length.argtypes = [C.c_double, C.c_double, _i64p]
        L.orc_create_edges_range.argtypes = [_dp, _i64, C.c_double, _i64, _i64, _u64, _u32p, _i64,
                                             _i64p, _i64p, _u64p]
        L.orc_create_edges.argtypes = [_dp, _i64, C.c_double, _i64p, _i64, _u64, _u32p, _i64, _i64p,
                                       _u64p]
        L.orc_edge_counts.argtypes = [_dp, _i64, C.c_double, _i64, _i64, _u64, _i64p]
        L.orc_node_cost.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.orc_block_bounds.argtypes = [_i64, C.c_int, C.c_int, _i64p, _i64p]
        L.orc_partition_of.argtypes = [C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int)]
        L.orc_block_cumulative.restype = C.c_double
        L.orc_block_cumulative.argtypes = [_dp, _i64, C.c_double, C.c_int, C.c_int, C.c_double, _dp]
        L.orc_plan_ucp.argtypes = [_dp, _i64, C.c_double, C.c_int, _i64p, _dp, _dp, _dp]

    def mix64(self, z: int) -> int:
        return self.lib.orc_mix64(z & 0xFFFFFFFFFFFFFFFF)

    def stream_open01(self, seed: int, u: int, count: int) -> np.ndarray:
        out = np.empty(count, np.float64)
        self.lib.orc_stream_open01(seed, u, count, _ptr(out, _dp))
        return out

    def blocked_sum(self, w) -> float:
        w = _f64(w)
        return self.lib.orc_blocked_sum(_ptr(w, _dp), w.size)

    def expected_total_edges(self, w, S: float) -> float:
        w = _f64(w)
        return self.lib.orc_expected_total_edges(_ptr(w, _dp), w.size, S)

    def synth_powerlaw(self, n, gamma, w_min, w_max, seed) -> np.ndarray:
        out = np.empty(n, np.float64)
        if self.lib.orc_synth_powerlaw(n, gamma, w_min, w_max, seed, _ptr(out, _dp)) != 0:
            raise OracleError("synth_powerlaw: bad arguments")
        return out

    def skip_length(self, p: float, r: float) -> int:
        out = _i64()
        if self.lib.orc_skip_length(p, r, C.byref(out)) != 0:
            raise OracleError("skip_length: p must be in (0,1] and r in (0,1)")
        return out.value

    def create_edges_range(self, w, S, lo, hi, seed, materialise=True, degree=False, cap=None):
        """Returns (pairs uint32[m,2] | None, count, checksum, degree int64[n] | None)."""
        w = _f64(w)
        cnt, cks = _i64(), _u64()
        pairs = None
        if materialise:
            if cap is None:
                self.lib.orc_create_edges_range(_ptr(w, _dp), w.size, S, lo, hi, seed, None, 0,
                                                None, C.byref(cnt), C.byref(cks))
                cap = cnt.value
            pairs = np.empty((max(cap, 1), 2), np.uint32)
        deg = np.zeros(w.size, np.int64) if degree else None
        rc = self.lib.orc_create_edges_range(_ptr(w, _dp), w.size, S, lo, hi, seed,
                                             _ptr(pairs, _u32p), cap or 0, _ptr(deg, _i64p),
                                             C.byref(cnt), C.byref(cks))
        if rc != 0:
            raise OracleError("create_edges_range: bad node range")
        if pairs is not None:
            pairs = pairs[: min(cnt.value, cap)]
        return pairs, cnt.value, cks.value, deg

    def create_edges(self, w, S, sources, seed, materialise=True):
        w = _f64(w)
        src = np.ascontiguousarray(sources, np.int64)
        cnt, cks = _i64(), _u64()
        rc = self.lib.orc_create_edges(_ptr(w, _dp), w.size, S, _ptr(src, _i64p), src.size, seed,
                                       None, 0, C.byref(cnt), C.byref(cks))
        if rc != 0:
            raise OracleError("create_edges: source node out of range")
        pairs = None
        if materialise:
            pairs = np.empty((max(cnt.value, 1), 2), np.uint32)
            self.lib.orc_create_edges(_ptr(w, _dp), w.size, S, _ptr(src, _i64p), src.size, seed,
                                      _ptr(pairs, _u32p), cnt.value, C.byref(cnt), C.byref(cks))
            pairs = pairs[: cnt.value]
        return pairs, cnt.value, cks.value

    def edge_counts(self, w, S, lo, hi, seed) -> np.ndarray:
        w = _f64(w)
        out = np.empty(hi - lo, np.int64)
        self.lib.orc_edge_counts(_ptr(w, _dp), w.size, S, lo, hi, seed, _ptr(out, _i64p))
        return out

    def node_cost(self, w, sigma, S) -> float:
        out = C.c_double()
        if self.lib.orc_node_cost(w, sigma, S, C.byref(out)) != 0:
            raise OracleError("node_cost: S must be > 0")
        return out.value

    def block_bounds(self, n, P, rank):
        lo, hi = _i64(), _i64()
        if self.lib.orc_block_bounds(n, P, rank, C.byref(lo), C.byref(hi)) != 0:
            raise OracleError("block_bounds: bad rank/P")
        return lo.value, hi.value

    def partition_of(self, c, z_bar, P) -> int:
        out = C.c_int()
        if self.lib.orc_partition_of(c, z_bar, P, C.byref(out)) != 0:
            raise OracleError("partition_of: Z_bar must be > 0")
        return out.value

    def block_cumulative(self, w, S, rank, P, sigma_start):
        w = _f64(w)
        lo, hi = self.block_bounds(w.size, P, rank)
        out = np.empty(max(hi - lo, 1), np.float64)
        bc = self.lib.orc_block_cumulative(_ptr(w, _dp), w.size, S, rank, P, sigma_start,
                                           _ptr(out, _dp))
        return out[: hi - lo], bc

    def plan_ucp(self, w, S, P, with_costs=False):
        """plan_ucp_oracle: boundaries int64[P+1] (+ C_u, block weights, block costs)."""
        w = _f64(w)
        if P < 1:
            raise OracleError("plan_ucp_oracle: P must be >= 1")
        b = np.empty(P + 1, np.int64)
        cum = np.empty(max(w.size, 1), np.float64) if with_costs else None
        bw = np.empty(P, np.float64)
        bc = np.empty(P, np.float64)
        self.lib.orc_plan_ucp(_ptr(w, _dp), w.size, S, P, _ptr(b, _i64p), _ptr(cum, _dp),
                              _ptr(bw, _dp), _ptr(bc, _dp))
        if with_costs:
            return b, cum[: w.size], bw, bc
        return b


# --------------------------------------------------------------------------- ref
class RefWS:
    """Owning handle on a reference clgen::WeightSequence."""

    def __init__(self, lib, handle):
        self._lib, self.h = lib, handle

    def __del__(self):
        try:
            self._lib.ref_ws_destroy(self.h)
        except Exception:
            pass

    @property
    def n(self) -> int:
        return self._lib.ref_ws_size(self.h)

    @property
    def sum_S(self) -> float:
        return self._lib.ref_ws_sum(self.h)

    @property
    def weights(self) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        self._lib.ref_ws_weights(self.h, _ptr(out, _dp))
        return out

    @property
    def labels(self) -> np.ndarray:
        out = np.empty(self.n, np.int64)
        self._lib.ref_ws_labels(self.h, _ptr(out, _i64p))
        return out


class _Ref:
    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference oracle not built: {path}")
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix64.restype = _u64
        L.ref_mix64.argtypes = [_u64]
        L.ref_stream_open01.argtypes = [_u64, _i64, _i64, _dp]
        L.ref_blocked_sum.argtypes = [_dp, _i64, _dp]
        L.ref_ws_create.argtypes = [_dp, _i64, C.c_int, C.POINTER(vp)]
        L.ref_ws_destroy.argtypes = [vp]
        L.ref_ws_sum.restype = C.c_double
        L.ref_ws_sum.argtypes = [vp]
        L.ref_ws_weights.argtypes = [vp, _dp]
        L.ref_ws_labels.argtypes = [vp, _i64p]
        L.ref_ws_size.restype = _i64
        L.ref_ws_size.argtypes = [vp]
        L.ref_synth_powerlaw.argtypes = [_i64, C.c_double, C.c_double, C.c_double, _u64,
                                         C.POINTER(vp)]
        L.ref_synth_constant.argtypes = [_i64, C.c_double, C.POINTER(vp)]
        L.ref_expected_total_edges.argtypes = [vp, _dp]
        L.ref_skip_length.argtypes = [C.c_double, C.c_double, _i64p]
        L.ref_node_cost.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.ref_block_bounds.argtypes = [_i64, C.c_int, C.c_int, _i64p, _i64p]
        L.ref_partition_of.argtypes = [C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int)]
        L.ref_create_edges_range.argtypes = [vp, C.c_double, _i64, _i64, _u64, _u32p, _i64, _i64p]
        L.ref_create_edges.argtypes = [vp, C.c_double, _i64p, _i64, _u64, _u32p, _i64, _i64p]
        L.ref_fold_edges_range.argtypes = [vp, C.c_double, _i64, _i64, _u64, _i64p, _i64p, _u64p]
        L.ref_naive_pair_sampler.argtypes = [vp, _u64, _u32p, _i64, _i64p]
        L.ref_plan_ucp_oracle.argtypes = [vp, C.c_int, _i64p]
        L.ref_node_costs_sequential.argtypes = [vp, _dp]
        L.ref_fill_partition_costs.argtypes = [vp, C.c_int, C.c_int, _i64p, _dp]
        L.ref_plan_ucp_spmd.argtypes = [vp, C.c_int, _i64p]
        L.ref_global_cum_costs.argtypes = [vp, C.c_int, _dp, _dp, _dp]
        L.ref_generate_count.argtypes = [vp, C.c_int, C.c_int, _u64, _i64p, _dp, _dp, _i64p]
        L.ref_parallel_ranges_count.argtypes = [vp, C.c_double, _i64p, C.c_int, _u64, _i64p, _dp]
        L.ref_write_edges.argtypes = [_u32p, _i64, C.c_int, C.c_char_p]
        L.ref_read_edges.argtypes = [C.c_char_p, _u32p, _i64, _i64p]
        L.ref_fidelity.argtypes = [vp, _u32p, _i64, C.c_double, _dp, C.POINTER(C.c_int), _dp, _i64p,
                                   _dp, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int)]

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(self.lib.ref_last_error().decode())

    def mix64(self, z: int) -> int:
        return self.lib.ref_mix64(z & 0xFFFFFFFFFFFFFFFF)

    def stream_open01(self, seed, u, count) -> np.ndarray:
        out = np.empty(count, np.float64)
        self.lib.ref_stream_open01(seed, u, count, _ptr(out, _dp))
        return out

    def blocked_sum(self, w) -> float:
        w = _f64(w)
        out = C.c_double()
        self._check(self.lib.ref_blocked_sum(_ptr(w, _dp), w.size, C.byref(out)))
        return out.value

    def weight_sequence(self, w, sort_desc: bool = False) -> RefWS:
        w = _f64(w)
        h = C.c_void_p()
        self._check(self.lib.ref_ws_create(_ptr(w, _dp), w.size, int(sort_desc), C.byref(h)))
        return RefWS(self.lib, h)

    def synth_powerlaw(self, n, gamma, w_min, w_max, seed) -> RefWS:
        h = C.c_void_p()
        self._check(self.lib.ref_synth_powerlaw(n, gamma, w_min, w_max, seed, C.byref(h)))
        return RefWS(self.lib, h)

    def synth_constant(self, n, d) -> RefWS:
        h = C.c_void_p()
        self._check(self.lib.ref_synth_constant(n, d, C.byref(h)))
        return RefWS(self.lib, h)

    def expected_total_edges(self, ws: RefWS) -> float:
        out = C.c_double()
        self._check(self.lib.ref_expected_total_edges(ws.h, C.byref(out)))
        return out.value

    def skip_length(self, p, r) -> int:
        out = _i64()
        self._check(self.lib.ref_skip_length(p, r, C.byref(out)))
        return out.value

    def node_cost(self, w, sigma, S) -> float:
        out = C.c_double()
        self._check(self.lib.ref_node_cost(w, sigma, S, C.byref(out)))
        return out.value

    def block_bounds(self, n, P, rank):
        lo, hi = _i64(), _i64()
        self._check(self.lib.ref_block_bounds(n, P, rank, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def partition_of(self, c, z_bar, P) -> int:
        out = C.c_int()
        self._check(self.lib.ref_partition_of(c, z_bar, P, C.byref(out)))
        return out.value

    def create_edges_range(self, ws: RefWS, S, lo, hi, seed, materialise=True):
        cnt = _i64()
        if not materialise:
            self._check(self.lib.ref_create_edges_range(ws.h, S, lo, hi, seed, None, 0,
                                                        C.byref(cnt)))
            return None, cnt.value
        self._check(self.lib.ref_create_edges_range(ws.h, S, lo, hi, seed, None, 0, C.byref(cnt)))
        pairs = np.empty((max(cnt.value, 1), 2), np.uint32)
        self._check(self.lib.ref_create_edges_range(ws.h, S, lo, hi, seed, _ptr(pairs, _u32p),
                                                    cnt.value, C.byref(cnt)))
        return pairs[: cnt.value], cnt.value

    def create_edges(self, ws: RefWS, S, sources, seed):
        src = np.ascontiguousarray(sources, np.int64)
        cnt = _i64()
        self._check(self.lib.ref_create_edges(ws.h, S, _ptr(src, _i64p), src.size, seed, None, 0,
                                              C.byref(cnt)))
        pairs = np.empty((max(cnt.value, 1), 2), np.uint32)
        self._check(self.lib.ref_create_edges(ws.h, S, _ptr(src, _i64p), src.size, seed,
                                              _ptr(pairs, _u32p), cnt.value, C.byref(cnt)))
        return pairs[: cnt.value], cnt.value

    def fold_edges_range(self, ws: RefWS, S, lo, hi, seed, degree=False):
        cnt, cks = _i64(), _u64()
        deg = np.zeros(ws.n, np.int64) if degree else None
        self._check(self.lib.ref_fold_edges_range(ws.h, S, lo, hi, seed, _ptr(deg, _i64p),
                                                  C.byref(cnt), C.byref(cks)))
        return cnt.value, cks.value, deg

    def naive_pair_sampler(self, ws: RefWS, seed):
        cnt = _i64()
        self._check(self.lib.ref_naive_pair_sampler(ws.h, seed, None, 0, C.byref(cnt)))
        pairs = np.empty((max(cnt.value, 1), 2), np.uint32)
        self._check(self.lib.ref_naive_pair_sampler(ws.h, seed, _ptr(pairs, _u32p), cnt.value,
                                                    C.byref(cnt)))
        return pairs[: cnt.value]

    def plan_ucp_oracle(self, ws: RefWS, P) -> np.ndarray:
        b = np.empty(max(P, 0) + 1, np.int64)
        self._check(self.lib.ref_plan_ucp_oracle(ws.h, P, _ptr(b, _i64p)))
        return b

    def node_costs_sequential(self, ws: RefWS) -> np.ndarray:
        out = np.empty(max(ws.n, 1), np.float64)
        self._check(self.lib.ref_node_costs_sequential(ws.h, _ptr(out, _dp)))
        return out[: ws.n]

    def fill_partition_costs(self, ws: RefWS, scheme: str, P: int, boundaries=None) -> np.ndarray:
        sch = {"naive": 0, "ucp": 1, "rrp": 2}[scheme]
        b = np.ascontiguousarray(boundaries if boundaries is not None else np.zeros(P + 1), np.int64)
        out = np.empty(P, np.float64)
        self._check(self.lib.ref_fill_partition_costs(ws.h, sch, P, _ptr(b, _i64p), _ptr(out, _dp)))
        return out

    def plan_ucp_spmd(self, ws: RefWS, P) -> np.ndarray:
        b = np.empty(P + 1, np.int64)
        self._check(self.lib.ref_plan_ucp_spmd(ws.h, P, _ptr(b, _i64p)))
        return b

    def global_cum_costs(self, ws: RefWS, P):
        cum = np.empty(max(ws.n, 1), np.float64)
        bw = np.empty(P, np.float64)
        bc = np.empty(P, np.float64)
        self._check(self.lib.ref_global_cum_costs(ws.h, P, _ptr(cum, _dp), _ptr(bw, _dp),
                                                  _ptr(bc, _dp)))
        return cum[: ws.n], bw, bc

    def generate_count(self, ws: RefWS, procs, seed, scheme="ucp"):
        sch = {"naive": 0, "ucp": 1, "rrp": 2}[scheme]
        tot, gen_ms, wall = _i64(), C.c_double(), C.c_double()
        b = np.zeros(procs + 1, np.int64)
        self._check(self.lib.ref_generate_count(ws.h, procs, sch, seed, C.byref(tot),
                                                C.byref(gen_ms), C.byref(wall), _ptr(b, _i64p)))
        return {"edges": tot.value, "gen_wall_ms": gen_ms.value, "wall_ms": wall.value,
                "boundaries": b}

    def write_edges(self, pairs, path: str, binary: bool = True) -> None:
        p = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
        self._check(self.lib.ref_write_edges(_ptr(p, _u32p), p.shape[0], int(binary),
                                             path.encode()))

    def read_edges(self, path: str) -> np.ndarray:
        cnt = _i64()
        self._check(self.lib.ref_read_edges(path.encode(), None, 0, C.byref(cnt)))
        out = np.empty((max(cnt.value, 1), 2), np.uint32)
        self._check(self.lib.ref_read_edges(path.encode(), _ptr(out, _u32p), cnt.value,
                                            C.byref(cnt)))
        return out[: cnt.value]

    def fidelity(self, ws: RefWS, pairs, flag_mass: float = 100.0) -> dict:
        """degree_histogram + compare_distributions (analysis.cpp:18-85)."""
        p = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
        cap = 128
        sc = np.zeros(5)
        k = np.zeros(cap, np.int32)
        ex = np.zeros(cap)
        gen = np.zeros(cap, np.int64)
        rel = np.zeros(cap)
        fl = np.zeros(cap, np.int32)
        nb = C.c_int()
        ip = C.POINTER(C.c_int)
        self._check(self.lib.ref_fidelity(ws.h, _ptr(p, _u32p), p.shape[0], flag_mass,
                                          _ptr(sc, _dp), k.ctypes.data_as(ip), _ptr(ex, _dp),
                                          _ptr(gen, _i64p), _ptr(rel, _dp), fl.ctypes.data_as(ip),
                                          cap, C.byref(nb)))
        m = min(nb.value, cap)
        return {"mean_expected": sc[0], "mean_generated": sc[1], "mean_rel_error": sc[2],
                "max_flagged_rel_error": sc[3], "zero_degree": int(sc[4]),
                "bins": [{"k": int(k[i]), "expected_count": float(ex[i]),
                          "generated_count": int(gen[i]), "rel_error": float(rel[i]),
                          "flagged": bool(fl[i])} for i in range(m)]}

    def parallel_ranges_count(self, ws: RefWS, S, ranges, seed):
        r = np.ascontiguousarray(ranges, np.int64).reshape(-1)
        tot, wall = _i64(), C.c_double()
        self._check(self.lib.ref_parallel_ranges_count(ws.h, S, _ptr(r, _i64p), r.size // 2, seed,
                                                       C.byref(tot), C.byref(wall)))
        return tot.value, wall.value


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)
