"""ctypes binding of the C ABI in ``include/clgen_dev.h`` (libclgen_b200.so).

There is no fallback: if the sm_100a library is missing or cannot be loaded,
importing the package's device API raises.  Build it with
``python -m paper_1406_1215_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CLGEN_LIB") or os.path.join(HERE, "libclgen_b200.so")  # CLGEN_LIB: A/B tooling only

CLGEN_OK = 0
CLGEN_EINVAL = -1
CLGEN_ECUDA = -2
CLGEN_ENOMEM = -3
CLGEN_ERANGE = -4

STREAM_REFERENCE = 0
STREAM_COUNTER = 1


class error(RuntimeError):
    """Contract violation or device failure (mirrors ``clgen::error``, types.hpp:11-13)."""

    def __init__(self, msg: str, code: int = CLGEN_EINVAL):
        super().__init__(msg)
        self.code = code


_lib = None
_lock = threading.Lock()

_i64 = C.c_int64
_u64 = C.c_uint64
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)


def _declare(L):
    L.clgen_dev_last_error.restype = C.c_char_p
    L.clgen_dev_version.restype = C.c_char_p
    L.clgen_dev_create.argtypes = [C.c_int, C.POINTER(_vp)]
    L.clgen_dev_destroy.argtypes = [_vp]
    L.clgen_dev_stream.restype = _vp
    L.clgen_dev_stream.argtypes = [_vp]
    L.clgen_dev_synchronize.argtypes = [_vp]
    L.clgen_dev_launch_count.restype = C.c_ulonglong
    L.clgen_dev_launch_count.argtypes = [_vp]
    L.clgen_dev_last_kernel_ms.argtypes = [_vp, C.POINTER(C.c_float)]
    L.clgen_dev_set_weights.argtypes = [_vp, _vp, _i64]
    L.clgen_dev_prefetch_weights.argtypes = [_vp, _vp, _i64]
    L.clgen_dev_num_nodes.restype = _i64
    L.clgen_dev_num_nodes.argtypes = [_vp]
    L.clgen_dev_weights.restype = _vp
    L.clgen_dev_weights.argtypes = [_vp]
    L.clgen_dev_device.argtypes = [_vp]
    L.clgen_dev_sort_desc.argtypes = [_vp, _vp, _i64, _vp]
    L.clgen_dev_copy_weights.argtypes = [_vp, _vp, _i64]
    L.clgen_dev_blocked_sum.argtypes = [_vp, _dp]
    L.clgen_dev_blocked_sum_array.argtypes = [_vp, _vp, _i64, _dp]
    L.clgen_dev_synth_powerlaw.argtypes = [_vp, _i64, C.c_double, C.c_double, C.c_double, _u64, C.c_int,
                                           C.c_double, _vp, _i64p]
    L.clgen_dev_create_edges_range.argtypes = [_vp, C.c_double, _i64, _i64, _u64, _vp, _i64, _i64p,
                                               _i64p]
    L.clgen_dev_create_edges.argtypes = [_vp, C.c_double, _vp, _i64, _u64, _vp, _i64, _i64p, _i64p]
    L.clgen_dev_edge_counts.argtypes = [_vp, C.c_double, _i64, _i64, _u64, _vp, _i64p, _i64p]
    L.clgen_dev_stream_range.argtypes = [_vp, C.c_double, _i64, _i64, _u64, C.c_int, C.c_int, _vp,
                                         C.c_int, _vp, _i64, _i64p, _u64p, _i64p]
    L.clgen_dev_flagged_nodes.argtypes = [_vp, _i64p, _i64, _i64p]
    L.clgen_dev_write_edges.argtypes = [_vp, _vp, _i64, C.c_int, C.c_char_p]
    _ip = C.POINTER(C.c_int)
    L.clgen_dev_fidelity.argtypes = [_vp, _vp, _i64, C.c_double, _dp, _ip, _dp, _i64p, _dp, _ip,
                                     C.c_int, _ip]
    L.clgen_dev_edge_degrees.argtypes = [_vp, _vp, _i64, _vp]
    L.clgen_dev_generate_range.argtypes = [_vp, C.c_double, _i64, _i64, _u64, C.c_int, _vp, _i64,
                                           _i64p, _i64p]
    L.clgen_dev_node_costs.argtypes = [_vp, _vp]
    L.clgen_dev_partition_costs.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp]
    L.clgen_dev_expected_total_edges.argtypes = [_vp, _dp]
    L.clgen_spmd_generate.argtypes = [_vp, C.c_int, _vp, _i64, _u64, C.c_int, _vp, _vp, _vp, _vp, _vp]
    L.clgen_dev_pair_trials.argtypes = [_vp, C.c_double, _u64, _i64, _vp]
    L.clgen_dev_set_counter_params.argtypes = [_vp, C.c_double, C.c_double]
    L.clgen_dev_set_fast_math.argtypes = [_vp, C.c_int]
    L.clgen_dev_set_warp_profile.argtypes = [_vp, C.c_int]
    L.clgen_dev_set_kernel_shape.argtypes = [_vp, C.c_int, C.c_int]
    L.clgen_dev_warp_profile.argtypes = [_vp, C.c_int, _dp, _dp, _dp, _dp, _i64p]
    L.clgen_dev_warp_profile_launches.argtypes = [_vp]
    L.clgen_dev_counter_plan_info.argtypes = [_vp, C.POINTER(C.c_int), _i64p, _i64p,
                                              C.POINTER(C.c_int), _dp]
    L.clgen_dev_plan_ucp.argtypes = [_vp, C.c_int, _vp, _vp]
    L.clgen_dev_plan_block_weight.argtypes = [_vp, C.c_int, C.c_int, _dp]
    L.clgen_dev_plan_block_costs.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double, _dp]
    L.clgen_dev_plan_block_boundaries.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double,
                                                  _vp]
    return L


# Every symbol include/clgen_dev.h declares (checked by the CPU test suite).
EXPORTS = (
    "clgen_dev_last_error", "clgen_dev_version", "clgen_dev_create", "clgen_dev_destroy",
    "clgen_dev_stream", "clgen_dev_synchronize", "clgen_dev_launch_count",
    "clgen_dev_last_kernel_ms", "clgen_dev_set_weights", "clgen_dev_prefetch_weights", "clgen_dev_num_nodes",
    "clgen_dev_weights", "clgen_dev_device", "clgen_dev_copy_weights", "clgen_dev_blocked_sum", "clgen_dev_blocked_sum_array", "clgen_dev_synth_powerlaw", "clgen_dev_sort_desc", "clgen_dev_create_edges_range",
    "clgen_dev_create_edges", "clgen_dev_edge_counts", "clgen_dev_stream_range",
    "clgen_dev_flagged_nodes", "clgen_dev_plan_ucp", "clgen_dev_plan_block_weight",
    "clgen_dev_plan_block_costs", "clgen_dev_plan_block_boundaries", "clgen_dev_generate_range",
    "clgen_dev_set_counter_params", "clgen_dev_pair_trials", "clgen_dev_counter_plan_info", "clgen_dev_set_fast_math",
    "clgen_dev_set_warp_profile", "clgen_dev_set_kernel_shape", "clgen_dev_warp_profile",
    "clgen_dev_warp_profile_launches", "clgen_dev_write_edges",
    "clgen_dev_fidelity", "clgen_dev_edge_degrees", "clgen_spmd_generate",
    "clgen_dev_node_costs", "clgen_dev_partition_costs", "clgen_dev_expected_total_edges",
)


def lib():
    """Load libclgen_b200.so (raises if it is absent: there is no CPU path)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} not built; run `python -m paper_1406_1215_b200.build` "
                        "(the generator has no CPU fallback)")
                _lib = _declare(C.CDLL(LIB_PATH))
    return _lib


def check(rc: int) -> None:
    if rc != CLGEN_OK:
        raise error(lib().clgen_dev_last_error().decode(), rc)
