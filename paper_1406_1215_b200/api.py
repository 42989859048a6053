"""Python mirror of the reference generator API (namespace clgen), backed by
the sm_100a library through the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/clgen/{weights,edge_skip}.hpp so parity
tests read like the reference's own tests:

=========================  ==================================================
this module                reference
=========================  ==================================================
``WeightSequence``         ``WeightSequence`` (weights.hpp:14-20)
``make_weight_sequence``   ``make_weight_sequence`` (weights.cpp:32-55)
``blocked_sum``            ``blocked_sum`` (weights.cpp:21-30)
``create_edges_range``     ``create_edges_range`` (edge_skip.cpp:60-66)
``create_edges``           ``create_edges`` (edge_skip.cpp:50-58)
``serial_cl``              ``serial_cl`` (edge_skip.cpp:68-70)
``stream_range``           streaming fold (no reference counterpart; the
                           count-only ``EdgeCounter`` sink generalised)
=========================  ==================================================

Edges are returned as ``uint32[m, 2]`` (u, v) pairs — the device layout; the
reference's ``Edge`` is two int64 (edge_skip.hpp:15-18), widen with
``.astype(np.int64)`` when comparing.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from ._lib import STREAM_COUNTER, STREAM_REFERENCE, check, error

try:  # torch is plumbing only: device buffers and streams
    import torch
except Exception:  # pragma: no cover
    torch = None


class SortPolicy(Enum):
    require_sorted = 0
    sort_desc = 1


def _addr(x) -> int:
    """Raw pointer of a numpy array or torch tensor (host or device)."""
    if x is None:
        return 0
    if torch is not None and isinstance(x, torch.Tensor):
        if not x.is_contiguous():
            raise error("tensor must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise error("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError(f"unsupported buffer type {type(x)!r}")


class Device:
    """One ``clgen_dev_ctx``: a CUDA device, its stream and resident weights."""

    def __init__(self, device: int = 0):
        L = _lib.lib()
        h = C.c_void_p()
        check(L.clgen_dev_create(int(device), C.byref(h)))
        self._h = h
        self.index = int(device)
        self._stream = None

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().clgen_dev_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def stream_ptr(self) -> int:
        return _lib.lib().clgen_dev_stream(self._h)

    def torch_stream(self):
        """The context stream as a torch stream (for CUDA-event timing)."""
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.stream_ptr, device=f"cuda:{self.index}")
        return self._stream

    def synchronize(self) -> None:
        check(_lib.lib().clgen_dev_synchronize(self._h))

    @property
    def launch_count(self) -> int:
        """Kernels launched by this context so far."""
        return int(_lib.lib().clgen_dev_launch_count(self._h))

    def last_kernel_ms(self) -> float:
        """Device time of the last sampler kernel (CUDA events on the context stream)."""
        ms = C.c_float()
        check(_lib.lib().clgen_dev_last_kernel_ms(self._h, C.byref(ms)))
        return ms.value

    def set_weights(self, w) -> None:
        if isinstance(w, np.ndarray):
            w = np.ascontiguousarray(w, np.float64)
        elif torch is not None and isinstance(w, torch.Tensor):
            if w.dtype != torch.float64:
                raise error("weights must be float64")
            w = w.contiguous()
        n = int(w.shape[0]) if w is not None else 0
        check(_lib.lib().clgen_dev_set_weights(self._h, _addr(w) if n else None, n))

    def prefetch_weights(self, w) -> None:
        """Start copying the NEXT weight array on the context's copy stream
        (overlaps the running generation); the next ``set_weights`` call with
        the same array takes that copy.  ``w`` must stay unchanged until then."""
        if isinstance(w, np.ndarray):
            if w.dtype != np.float64 or not w.flags["C_CONTIGUOUS"]:
                raise error("prefetch_weights: contiguous float64 array required")
        elif torch is not None and isinstance(w, torch.Tensor):
            if w.dtype != torch.float64 or not w.is_contiguous():
                raise error("prefetch_weights: contiguous float64 tensor required")
        check(_lib.lib().clgen_dev_prefetch_weights(self._h, _addr(w), int(w.shape[0])))

    @property
    def n(self) -> int:
        return int(_lib.lib().clgen_dev_num_nodes(self._h))

    def weights_tensor(self):
        """Zero-copy torch view of the resident weights (float64, device)."""
        ptr = _lib.lib().clgen_dev_weights(self._h)
        n = self.n
        if n == 0:
            return torch.empty(0, dtype=torch.float64, device=f"cuda:{self.index}")
        return _device_view(ptr, n, torch.float64, self.index)

    def blocked_sum(self) -> float:
        out = C.c_double()
        check(_lib.lib().clgen_dev_blocked_sum(self._h, C.byref(out)))
        return out.value

    def set_counter_params(self, class_eps: float = 0.0, chunk_cand: float = 0.0) -> None:
        """Counter-stream weight-class width and chunk size in expected
        candidates (0: automatic, a function of the weights); part of the
        stream definition (changes the graph, not its law)."""
        check(_lib.lib().clgen_dev_set_counter_params(self._h, class_eps, chunk_cand))

    def set_fast_math(self, enable: bool = True) -> None:
        """Reference-stream arithmetic: guarded fast path (default) or the
        reference expressions everywhere; both give identical edges."""
        check(_lib.lib().clgen_dev_set_fast_math(self._h, int(bool(enable))))

    def set_kernel_shape(self, shape: int = -1, heavy_phase: bool = True) -> None:
        """Kernel schedule: counter-stream shape (256 threads x 2/3/4/5/6 CTAs
        per SM for shape 0/1/2/3/4; -1: default 1) and whether the reference
        stream walks its heaviest chains one per warp; the edge set does not
        depend on either."""
        check(_lib.lib().clgen_dev_set_kernel_shape(self._h, int(shape), 0 if heavy_phase else 1))

    def set_warp_profile(self, enable: bool = True) -> None:
        check(_lib.lib().clgen_dev_set_warp_profile(self._h, int(bool(enable))))

    def warp_profile(self) -> list:
        """Per sampler launch of the last generation call: max/mean per-warp busy
        time (level-2 balance), mean/max ms, span ms, warps."""
        L = _lib.lib()
        out = []
        for i in range(L.clgen_dev_warp_profile_launches(self._h)):
            r, mean, mx, span = C.c_double(), C.c_double(), C.c_double(), C.c_double()
            k = C.c_int64()
            check(L.clgen_dev_warp_profile(self._h, i, C.byref(r), C.byref(mean), C.byref(mx),
                                           C.byref(span), C.byref(k)))
            out.append({"max_over_mean": r.value, "mean_ms": mean.value, "max_ms": mx.value,
                        "span_ms": span.value, "warps": k.value})
        return out

    def counter_plan_info(self) -> dict:
        """Counter plan of the last counter-stream call: classes, class-pair
        blocks, chunks over all sources, dense blocks, class width used."""
        k, b, ch, dn, eps = C.c_int(), C.c_int64(), C.c_int64(), C.c_int(), C.c_double()
        check(_lib.lib().clgen_dev_counter_plan_info(self._h, C.byref(k), C.byref(b), C.byref(ch),
                                                     C.byref(dn), C.byref(eps)))
        return {"classes": k.value, "blocks": b.value, "chunks": ch.value,
                "dense_blocks": dn.value, "class_eps": eps.value}

    def flagged_nodes(self) -> np.ndarray:
        n = C.c_int64()
        buf = np.empty(4096, np.int64)
        check(_lib.lib().clgen_dev_flagged_nodes(self._h, buf.ctypes.data_as(C.POINTER(C.c_int64)),
                                                 buf.size, C.byref(n)))
        return buf[: min(n.value, buf.size)]


def _device_view(ptr: int, n: int, dtype, device: int):
    """Wrap a raw device pointer owned by the library as a torch tensor (no copy)."""
    itemsize = torch.empty((), dtype=dtype).element_size()

    class _Holder:
        __cuda_array_interface__ = {
            "shape": (n,),
            "typestr": {torch.float64: "<f8", torch.int64: "<i8", torch.uint32: "<u4"}[dtype],
            "data": (ptr, True),
            "version": 3,
        }

    del itemsize
    with torch.cuda.device(device):
        return torch.as_tensor(_Holder(), device=f"cuda:{device}")


_default_devices: dict[int, Device] = {}


def default_device(index: int = 0) -> Device:
    if index not in _default_devices:
        _default_devices[index] = Device(index)
    return _default_devices[index]


@dataclass
class WeightSequence:
    """Sorted non-increasing weights resident on one GPU (weights.hpp:14-20).

    ``weights`` is the host copy (float64), ``sum_S`` the canonical
    ``blocked_sum`` computed on the device, ``orig_labels`` the permutation
    back to input order.  ``device`` owns the device copy.
    """

    weights: np.ndarray
    sum_S: float
    orig_labels: np.ndarray
    device: Device = field(repr=False)

    def size(self) -> int:
        return int(self.weights.shape[0])

    @property
    def n(self) -> int:
        return self.size()


def make_weight_sequence(weights, policy: SortPolicy = SortPolicy.require_sorted,
                         device: Device | int | None = None) -> WeightSequence:
    """weights.cpp:32-55.  ``sort_desc`` is a stable descending sort with labels;
    ``require_sorted`` raises ``error("weights unsorted at position u")``."""
    # each sequence owns its context unless one is passed in explicitly
    dev = device if isinstance(device, Device) else Device(device or 0)
    w = np.ascontiguousarray(weights, np.float64).reshape(-1)
    labels = np.arange(w.size, dtype=np.int64)
    if policy == SortPolicy.sort_desc:
        labels = np.argsort(-w, kind="stable").astype(np.int64)
        w = np.ascontiguousarray(w[labels])
    dev.set_weights(w)  # validates order on the device
    S = dev.blocked_sum()
    return WeightSequence(w, S, labels, dev)


def synth_powerlaw_device(n: int, gamma: float, w_min: float, w_max: float, seed: int,
                          device: Device | int | None = None, sort: bool = True,
                          target_mean: float = 0.0):
    """synth_powerlaw (weights.cpp:103-128) on the device, sorted descending
    (weights.cpp:32-55) unless ``sort`` is false: a float64 device tensor whose
    contents equal the reference's array bit for bit, and the number of draws
    the host's libm had to resolve.  ``target_mean`` > 0 rescales to that mean
    (the C4 recipe)."""
    if torch is None:
        raise RuntimeError("synth_powerlaw_device needs torch for the device buffer")
    dev = device if isinstance(device, Device) else default_device(device or 0)
    out = torch.empty(max(int(n), 1), dtype=torch.float64, device=f"cuda:{dev.index}")
    resolved = C.c_int64()
    check(_lib.lib().clgen_dev_synth_powerlaw(dev.handle, int(n), float(gamma), float(w_min), float(w_max),
                                              seed & 0xFFFFFFFFFFFFFFFF, 1 if sort else 0,
                                              float(target_mean), out.data_ptr(), C.byref(resolved)))
    return out[: max(int(n), 0)], resolved.value


def synth_powerlaw(n: int, gamma: float, w_min: float, w_max: float, seed: int,
                   device: Device | int | None = None, target_mean: float = 0.0) -> WeightSequence:
    """make_weight_sequence(synth_powerlaw(...)) with the weights synthesised,
    sorted and kept on the device (one device-to-host copy for ``.weights``)."""
    dev = device if isinstance(device, Device) else Device(device or 0)
    L = _lib.lib()
    # d_out = NULL: synthesised into scratch and installed as the context's weights
    check(L.clgen_dev_synth_powerlaw(dev.handle, int(n), float(gamma), float(w_min), float(w_max),
                                     seed & 0xFFFFFFFFFFFFFFFF, 1, float(target_mean), None, None))
    w = np.empty(int(n), np.float64)
    check(L.clgen_dev_copy_weights(dev.handle, w.ctypes.data, int(n)))
    return WeightSequence(w, dev.blocked_sum(), np.arange(w.size, dtype=np.int64), dev)


def sort_desc_device(w, device: Device | int | None = None):
    """SortPolicy.sort_desc (weights.cpp:32-55) on the device: sorts the float64
    device tensor ``w`` in place (stable, non-increasing) and returns
    ``(w, orig_labels)`` with the labels as an int64 device tensor."""
    if torch is None or not isinstance(w, torch.Tensor) or not w.is_cuda or w.dtype != torch.float64:
        raise error("sort_desc_device: float64 device tensor required")
    dev = device if isinstance(device, Device) else default_device(device or w.device.index or 0)
    labels = torch.empty(w.numel(), dtype=torch.int64, device=w.device)
    check(_lib.lib().clgen_dev_sort_desc(dev.handle, _addr(w), int(w.numel()), labels.data_ptr()))
    return w, labels


def synth_constant(n: int, d: float, device: Device | int | None = None) -> WeightSequence:
    """weights.cpp:130-140 (same contract errors)."""
    if n < 1:
        raise error("synth_constant: n must be >= 1")
    if d < 0.0:
        raise error("synth_constant: d must be >= 0")
    if d > 0.0 and d >= float(n):
        raise error(f"synth_constant: inadmissible (d^2 = {d * d:g} >= S = {d * n:g})")
    return make_weight_sequence(np.full(int(n), float(d)), SortPolicy.require_sorted, device)


@dataclass
class ValidationReport:
    """weights.hpp:22-29."""
    is_sorted: bool = False
    admissible: bool = False  # max w^2 < S; false when S == 0
    n: int = 0
    sum_S: float = 0.0
    max_weight: float = 0.0
    zero_weight_count: int = 0


def validate(ws: WeightSequence) -> ValidationReport:
    """weights.cpp:142-153 (host: O(n) input statistics)."""
    w = ws.weights
    rep = ValidationReport(n=int(w.size), sum_S=float(ws.sum_S))
    rep.is_sorted = bool(np.all(w[:-1] >= w[1:])) if w.size > 1 else True
    rep.max_weight = float(max(0.0, w.max())) if w.size else 0.0
    rep.zero_weight_count = int(np.count_nonzero(w == 0.0))
    rep.admissible = ws.sum_S > 0.0 and rep.max_weight * rep.max_weight < ws.sum_S
    return rep


def blocked_sum(xs, device: Device | int | None = None) -> float:
    """weights.cpp:21-30 on the device, for any sequence (host or device)."""
    dev = device if isinstance(device, Device) else default_device(device or 0)
    if isinstance(xs, np.ndarray) or not (torch is not None and isinstance(xs, torch.Tensor)):
        xs = np.ascontiguousarray(xs, np.float64).reshape(-1)
    out = C.c_double()
    n = int(xs.shape[0])
    check(_lib.lib().clgen_dev_blocked_sum_array(dev.handle, _addr(xs) if n else None, n,
                                                 C.byref(out)))
    return out.value


def _as_pairs(buf: np.ndarray, m: int) -> np.ndarray:
    return buf[:m]


def create_edges_range(ws: WeightSequence, S: float, lo: int, hi: int, seed: int,
                       out=None, return_flagged: bool = False):
    """edge_skip.cpp:60-66.  Returns ``uint32[m,2]`` (host) or fills ``out``
    (a device tensor of shape [cap,2], uint32/int32) and returns its prefix."""
    L = _lib.lib()
    cnt, nfl = C.c_int64(), C.c_int64()
    if out is None:
        # size with the count pass (cheap relative to materialisation)
        total = edge_total(ws, S, lo, hi, seed)
        buf = np.empty((max(total, 1), 2), np.uint32)
        check(L.clgen_dev_create_edges_range(ws.device.handle, S, lo, hi, seed & 0xFFFFFFFFFFFFFFFF,
                                             buf.ctypes.data, total, C.byref(cnt), C.byref(nfl)))
        res = buf[: cnt.value]
    else:
        cap = int(out.shape[0])
        rc = L.clgen_dev_create_edges_range(ws.device.handle, S, lo, hi, seed & 0xFFFFFFFFFFFFFFFF,
                                            _addr(out), cap, C.byref(cnt), C.byref(nfl))
        check(rc)
        res = out[: cnt.value]
    return (res, nfl.value) if return_flagged else res


def create_edges(ws: WeightSequence, S: float, sources, seed: int, return_flagged: bool = False):
    """edge_skip.cpp:50-58: sources walked in list order."""
    L = _lib.lib()
    src = np.ascontiguousarray(sources, np.int64).reshape(-1)
    cnt, nfl = C.c_int64(), C.c_int64()
    # first call with cap=0 learns the count (CLGEN_ERANGE when non-zero)
    rc = L.clgen_dev_create_edges(ws.device.handle, S, src.ctypes.data if src.size else None,
                                  src.size, seed & 0xFFFFFFFFFFFFFFFF, None, 0, C.byref(cnt),
                                  C.byref(nfl))
    if rc not in (_lib.CLGEN_OK, _lib.CLGEN_ERANGE):
        check(rc)
    total = cnt.value
    buf = np.empty((max(total, 1), 2), np.uint32)
    if total:
        check(L.clgen_dev_create_edges(ws.device.handle, S, src.ctypes.data, src.size,
                                       seed & 0xFFFFFFFFFFFFFFFF, buf.ctypes.data, total,
                                       C.byref(cnt), C.byref(nfl)))
    res = buf[: cnt.value]
    return (res, nfl.value) if return_flagged else res


def serial_cl(ws: WeightSequence, seed: int, return_flagged: bool = False):
    """edge_skip.cpp:68-70."""
    return create_edges_range(ws, ws.sum_S, 0, ws.size(), seed, return_flagged=return_flagged)


def edge_counts(ws: WeightSequence, S: float, lo: int, hi: int, seed: int) -> np.ndarray:
    """Count pass: per-source edge counts for [lo, hi)."""
    out = np.empty(max(hi - lo, 1), np.int32)
    tot, nfl = C.c_int64(), C.c_int64()
    check(_lib.lib().clgen_dev_edge_counts(ws.device.handle, S, lo, hi, seed & 0xFFFFFFFFFFFFFFFF,
                                           out.ctypes.data, C.byref(tot), C.byref(nfl)))
    return out[: hi - lo]


def edge_total(ws: WeightSequence, S: float, lo: int, hi: int, seed: int) -> int:
    tot, nfl = C.c_int64(), C.c_int64()
    check(_lib.lib().clgen_dev_edge_counts(ws.device.handle, S, lo, hi, seed & 0xFFFFFFFFFFFFFFFF,
                                           None, C.byref(tot), C.byref(nfl)))
    return tot.value


@dataclass
class StreamResult:
    count: int
    checksum: int
    flagged: int
    degree: object = None  # uint32 tracked degrees (numpy or the caller's tensor)


def stream_range(ws: WeightSequence, S: float, lo: int, hi: int, seed: int,
                 mode: str = "reference", track_shift: int | None = None, degree=None,
                 accumulate: bool = False, ring=None) -> StreamResult:
    """Streaming generation fused with the fold (edge count, 64-bit checksum
    sum mix64((u<<32)|v), tracked undirected degrees).  ``track_shift=None``
    disables degree tracking.  ``ring`` (device uint32 tensor [cap,2], cap a
    power of two) receives every edge at position mod cap."""
    L = _lib.lib()
    sm = {"reference": STREAM_REFERENCE, "counter": STREAM_COUNTER}[mode]
    cnt, cks, nfl = C.c_int64(), C.c_uint64(), C.c_int64()
    if track_shift is not None and degree is None:
        ntr = (ws.size() + (1 << track_shift) - 1) >> track_shift
        degree = np.zeros(max(ntr, 1), np.uint32)
    ring_cap = int(ring.shape[0]) if ring is not None else 0
    check(L.clgen_dev_stream_range(ws.device.handle, S, lo, hi, seed & 0xFFFFFFFFFFFFFFFF, sm,
                                   track_shift or 0, _addr(degree) if degree is not None else None,
                                   int(accumulate), _addr(ring) if ring is not None else None,
                                   ring_cap, C.byref(cnt), C.byref(cks), C.byref(nfl)))
    return StreamResult(cnt.value, cks.value, nfl.value, degree)


def node_costs_sequential(ws: WeightSequence) -> np.ndarray:
    """cost.cpp:62-77 on the device, bit-identical (float64[n])."""
    out = np.empty(max(ws.size(), 1), np.float64)
    check(_lib.lib().clgen_dev_node_costs(ws.device.handle, out.ctypes.data))
    return out[: ws.size()]


def fill_partition_costs(plan: "PartitionPlan", ws: WeightSequence) -> np.ndarray:
    """partition.cpp:205-222 on the device, bit-identical: per-partition
    expected cost (float64[P]); also stored as plan.per_partition_cost."""
    scheme = {"naive": 0, "ucp": 1, "rrp": 2}[plan.scheme]
    per = np.zeros(plan.procs, np.float64)
    b = None if plan.boundaries is None else np.ascontiguousarray(plan.boundaries, np.int64)
    check(_lib.lib().clgen_dev_partition_costs(ws.device.handle, scheme, plan.procs,
                                               b.ctypes.data if b is not None else None,
                                               per.ctypes.data))
    plan.per_partition_cost = per
    return per


def expected_total_edges(ws: WeightSequence) -> float:
    """weights.cpp:155-162 on the device, bit-identical."""
    out = C.c_double()
    check(_lib.lib().clgen_dev_expected_total_edges(ws.device.handle, C.byref(out)))
    return out.value


def pair_trials(ws: WeightSequence, S: float, seed: int, trials: int) -> np.ndarray:
    """Counter stream over all sources for seeds seed..seed+trials-1 in one
    launch; returns uint32[n, n] per-pair edge counts (n <= 4096)."""
    n = ws.size()
    out = np.zeros((n, n), np.uint32)
    check(_lib.lib().clgen_dev_pair_trials(ws.device.handle, S, seed & 0xFFFFFFFFFFFFFFFF, int(trials),
                                           out.ctypes.data))
    return out


class _SpmdReport(C.Structure):
    _fields_ = [("G", C.c_int), ("S", C.c_double), ("S_check", C.c_double),
                ("total_edges", C.c_int64), ("checksum", C.c_uint64), ("n_flagged", C.c_int64),
                ("wall_ms", C.c_double), ("plan_ms", C.c_double), ("nccl_version", C.c_int)]


def spmd_generate(weights, devices, seed: int, mode: str = "counter") -> dict:
    """generate(ws, GenConfig) over one host thread per GPU (runtime.cpp:93-138,
    comm.cpp:204-227): level-1 UCP plan with NCCL collectives, each rank
    streams its partition; returns the plan, per-rank counts/times and totals."""
    w = np.ascontiguousarray(weights, np.float64).reshape(-1)
    devs = np.ascontiguousarray(devices, np.int32).reshape(-1)
    G = int(devs.size)
    sm = {"reference": STREAM_REFERENCE, "counter": STREAM_COUNTER}[mode]
    b = np.zeros(G + 1, np.int64)
    edges = np.zeros(G, np.int64)
    gen_ms = np.zeros(G)
    kern_ms = np.zeros(G)
    rep = _SpmdReport()
    check(_lib.lib().clgen_spmd_generate(devs.ctypes.data, G, w.ctypes.data if w.size else None, w.size,
                                         seed & 0xFFFFFFFFFFFFFFFF, sm, b.ctypes.data, edges.ctypes.data,
                                         gen_ms.ctypes.data, kern_ms.ctypes.data, C.byref(rep)))
    return {"boundaries": b, "rank_edges": edges, "rank_gen_ms": gen_ms, "rank_kernel_ms": kern_ms,
            "G": rep.G, "S": rep.S, "S_check": rep.S_check, "total_edges": rep.total_edges,
            "checksum": rep.checksum, "n_flagged": rep.n_flagged, "wall_ms": rep.wall_ms,
            "plan_ms": rep.plan_ms, "nccl_version": rep.nccl_version}


def plan_ucp(ws: WeightSequence, P: int, with_costs: bool = False):
    """Level-1 UCP on the device, bit-identical to plan_ucp_oracle(ws, P)
    (partition.cpp:159-203).  Returns int64[P+1] boundaries, plus the
    finalized C_u (float64[n]) when ``with_costs``."""
    if P < 1:
        raise error("plan_ucp_oracle: P must be >= 1")
    b = np.empty(P + 1, np.int64)
    cum = np.empty(max(ws.size(), 1), np.float64) if with_costs else None
    check(_lib.lib().clgen_dev_plan_ucp(ws.device.handle, int(P), b.ctypes.data,
                                        cum.ctypes.data if with_costs else None))
    if with_costs:
        return b, cum[: ws.size()]
    return b


def generate_range(ws: WeightSequence, S: float, lo: int, hi: int, seed: int,
                   mode: str = "counter", out=None):
    """Materialised generation with either stream (uint32[m,2], u then v ascending)."""
    L = _lib.lib()
    sm = {"reference": STREAM_REFERENCE, "counter": STREAM_COUNTER}[mode]
    cnt, nfl = C.c_int64(), C.c_int64()
    if out is None:
        rc = L.clgen_dev_generate_range(ws.device.handle, S, lo, hi, seed & 0xFFFFFFFFFFFFFFFF, sm,
                                        None, 0, C.byref(cnt), C.byref(nfl))
        if rc not in (_lib.CLGEN_OK, _lib.CLGEN_ERANGE):
            check(rc)
        total = cnt.value
        buf = np.empty((max(total, 1), 2), np.uint32)
        if total:
            check(L.clgen_dev_generate_range(ws.device.handle, S, lo, hi, seed & 0xFFFFFFFFFFFFFFFF,
                                             sm, buf.ctypes.data, total, C.byref(cnt),
                                             C.byref(nfl)))
        return buf[: cnt.value]
    check(L.clgen_dev_generate_range(ws.device.handle, S, lo, hi, seed & 0xFFFFFFFFFFFFFFFF, sm,
                                     _addr(out), int(out.shape[0]), C.byref(cnt), C.byref(nfl)))
    return out[: cnt.value]


# ---- partitions other than UCP (partition.cpp:47-67) ----------------------
@dataclass
class PartitionPlan:
    """partition.hpp:20-31 (boundaries for naive/ucp; strided for rrp)."""
    scheme: str
    procs: int
    n: int
    boundaries: np.ndarray | None = None
    per_partition_cost: np.ndarray | None = None

    def partition_size(self, i: int) -> int:
        if i < 0 or i >= self.procs:
            raise error("partition_size: bad partition index")
        if self.scheme == "rrp":
            return (self.n - 1 - i) // self.procs + 1 if self.n > i else 0
        return int(self.boundaries[i + 1] - self.boundaries[i])

    def partition_nodes(self, i: int) -> np.ndarray:
        """Ascending source nodes owned by partition i (partition.cpp:36-45)."""
        if self.scheme == "rrp":
            return np.arange(i, self.n, self.procs, dtype=np.int64)
        return np.arange(self.boundaries[i], self.boundaries[i + 1], dtype=np.int64)


def plan_naive(n: int, P: int) -> PartitionPlan:
    """partition.cpp:47-57 (ceil-first blocks, cost.cpp:15-22)."""
    if P < 1:
        raise error("plan_naive: P must be >= 1")
    from .plan import block_bounds
    b = np.array([0] + [block_bounds(n, P, i)[1] for i in range(P)], np.int64)
    return PartitionPlan("naive", P, n, b)


def plan_rrp(n: int, P: int) -> PartitionPlan:
    """partition.cpp:59-67 (u mod P)."""
    if P < 1:
        raise error("plan_rrp: P must be >= 1")
    return PartitionPlan("rrp", P, n, None)


def plan(ws: WeightSequence, scheme: str, P: int) -> PartitionPlan:
    if scheme == "ucp":
        return PartitionPlan("ucp", P, ws.size(), plan_ucp(ws, P))
    if scheme == "naive":
        return plan_naive(ws.size(), P)
    if scheme == "rrp":
        return plan_rrp(ws.size(), P)
    raise error("unknown scheme: " + scheme)


def generate_partition(ws: WeightSequence, p: PartitionPlan, i: int, seed: int):
    """Partition i's edges, as generate_on_rank walks them (runtime.cpp:76-82)."""
    if p.scheme == "rrp":
        return create_edges(ws, ws.sum_S, p.partition_nodes(i), seed)
    return create_edges_range(ws, ws.sum_S, int(p.boundaries[i]), int(p.boundaries[i + 1]), seed)


# ---- edge files (edge_io.cpp) ---------------------------------------------
def write_edges(edges, path: str, fmt: str = "binary", device: Device | None = None) -> None:
    """edge_io.cpp:72-88; `edges` uint32[m,2] host array or device tensor."""
    if fmt not in ("binary", "bin", "text"):
        raise error("unknown edge format: " + fmt)
    dev = device or default_device(0)
    m = int(edges.shape[0])
    check(_lib.lib().clgen_dev_write_edges(dev.handle, _addr(edges) if m else None, m,
                                           int(fmt != "text"), path.encode()))


def read_edges(path: str) -> np.ndarray:
    """edge_io.cpp:90-123 (binary sniffed by magic, else text) -> uint32[m,2]."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:8] == b"CLGEDGE1":
        if len(data) < 24:
            raise error(f"{path}: truncated edge header")
        ver = int.from_bytes(data[8:12], "little")
        if ver != 1:
            raise error(f"{path}: unsupported edge file version {ver}")
        cnt = int.from_bytes(data[16:24], "little")
        body = np.frombuffer(data, dtype="<u8", offset=24)
        if body.size < 2 * cnt:
            raise error(f"{path}: truncated at record {body.size // 2} of {cnt}")
        return body[: 2 * cnt].reshape(-1, 2).astype(np.uint32)
    rows = []
    for lineno, line in enumerate(data.decode().splitlines(), 1):
        if not line or line[0] == "#":
            continue
        parts = line.split()
        if len(parts) < 2:
            raise error(f"{path}: malformed edge at line {lineno}")
        rows.append((int(parts[0]), int(parts[1])))
    return np.array(rows, np.uint32).reshape(-1, 2)


# ---- degree fidelity (analysis.cpp:18-85) ----------------------------------
def edge_degrees(ws: WeightSequence, edges) -> np.ndarray:
    """Undirected degrees (uint32[n]) of a materialised edge list."""
    out = np.zeros(max(ws.size(), 1), np.uint32)
    m = int(edges.shape[0])
    check(_lib.lib().clgen_dev_edge_degrees(ws.device.handle, _addr(edges) if m else None, m,
                                            out.ctypes.data))
    return out[: ws.size()]


def fidelity(ws: WeightSequence, degree, total_edges: int, flag_mass: float = 100.0) -> dict:
    """compare_distributions(ws, degree_histogram(edges)) on the device."""
    cap = 256
    sc = np.zeros(5)
    k = np.zeros(cap, np.int32)
    ex = np.zeros(cap)
    gen = np.zeros(cap, np.int64)
    rel = np.zeros(cap)
    fl = np.zeros(cap, np.int32)
    nb = C.c_int()
    if isinstance(degree, np.ndarray):
        degree = np.ascontiguousarray(degree, np.uint32)
    ip = C.POINTER(C.c_int)
    check(_lib.lib().clgen_dev_fidelity(ws.device.handle, _addr(degree), int(total_edges),
                                        float(flag_mass), sc.ctypes.data_as(C.POINTER(C.c_double)),
                                        k.ctypes.data_as(ip),
                                        ex.ctypes.data_as(C.POINTER(C.c_double)),
                                        gen.ctypes.data_as(C.POINTER(C.c_int64)),
                                        rel.ctypes.data_as(C.POINTER(C.c_double)),
                                        fl.ctypes.data_as(ip), cap, C.byref(nb)))
    m = min(nb.value, cap)
    return {"mean_expected": sc[0], "mean_generated": sc[1], "mean_rel_error": sc[2],
            "max_flagged_rel_error": sc[3], "zero_degree": int(sc[4]),
            "bins": [{"k": int(k[i]), "expected_count": float(ex[i]),
                      "generated_count": int(gen[i]), "rel_error": float(rel[i]),
                      "flagged": bool(fl[i])} for i in range(m)]}
