"""Level-1 UCP plan across GPUs (partition.cpp:107-157, plan_ucp).

Each rank runs the device phases on its own rank block and the host performs
the reference's collectives with torch.distributed (NCCL over NVLink on the
GPU box, gloo in the CPU tests):

=====================================  ========================================
reference (in-process Communicator)    here
=====================================  ========================================
all_reduce_sum(block_weight)           all_gather(block weights) + rank-ordered
  runtime.cpp:55-58 (sum check)          fold (bit-identical to comm.cpp:39-45)
exclusive_scan_sum(block_weight) :117  same gather, fold of ranks < g
exclusive_scan_sum(block_cost)   :120  all_gather(block costs) + ordered fold
all_reduce_sum(block_cost)       :123  fold of all gathered block costs
send/recv_boundary + all_gather  :134  all_reduce(MIN) of each rank's found
                                        boundaries (n where none)
=====================================  ========================================

Never let the collective itself add FP64 values: NCCL's reduction order is not
the reference's, so doubles are gathered and folded on the host in rank order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check


def fold_prefix(xs, count: int) -> float:
    """partition.cpp:83-87 / comm.cpp:47-53: left fold from 0.0 of xs[:count]."""
    acc = 0.0
    for j in range(count):
        acc += float(xs[j])
    return acc


def block_bounds(n: int, P: int, rank: int) -> tuple[int, int]:
    """cost.cpp:15-22."""
    if P < 1 or rank < 0 or rank >= P:
        raise _lib.error("block_bounds: bad rank/P")
    q, r = divmod(n, P)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


class DevicePhases:
    """The per-rank device phases through the C ABI."""

    def __init__(self, dev):
        self.dev = dev

    def block_weight(self, G: int, g: int) -> float:
        out = C.c_double()
        check(_lib.lib().clgen_dev_plan_block_weight(self.dev.handle, G, g, C.byref(out)))
        return out.value

    def block_costs(self, G: int, g: int, sigma_start: float, S: float) -> float:
        out = C.c_double()
        check(_lib.lib().clgen_dev_plan_block_costs(self.dev.handle, G, g, sigma_start, S,
                                                    C.byref(out)))
        return out.value

    def block_boundaries(self, G: int, g: int, z_offset: float, z_bar: float) -> np.ndarray:
        found = np.empty(G + 1, np.int64)
        check(_lib.lib().clgen_dev_plan_block_boundaries(self.dev.handle, G, g, z_offset, z_bar,
                                                         found.ctypes.data))
        return found


@dataclass
class PlanResult:
    boundaries: np.ndarray   # int64[G+1]
    reduced_sum: float       # rank-ordered fold of block weights (runtime.cpp:55-58)
    block_weights: np.ndarray
    block_costs: np.ndarray
    z_bar: float


class TorchComm:
    """The two collectives the plan needs, on torch.distributed."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.device = device  # torch device for NCCL tensors, None for gloo (CPU)

    def all_gather_f64(self, x: float) -> np.ndarray:
        t = self.torch
        v = t.tensor([x], dtype=t.float64, device=self.device)
        out = t.empty(self.dist.get_world_size(), dtype=t.float64, device=self.device)
        self.dist.all_gather_into_tensor(out, v)
        return out.cpu().numpy()

    def all_reduce_min_i64(self, xs: np.ndarray) -> np.ndarray:
        t = self.torch
        v = t.from_numpy(np.ascontiguousarray(xs, np.int64)).to(self.device or "cpu")
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MIN)
        return v.cpu().numpy()


def plan_ucp_collective(phases, n: int, S: float, G: int, g: int, comm) -> PlanResult:
    """partition.cpp:107-157 for rank g of G: device phases + ordered host folds."""
    if n == 0:
        return PlanResult(np.zeros(G + 1, np.int64), 0.0, np.zeros(G), np.zeros(G), 0.0)
    bw = phases.block_weight(G, g)
    bws = comm.all_gather_f64(bw)
    sigma_start = fold_prefix(bws, g)
    z = phases.block_costs(G, g, sigma_start, S)
    zs = comm.all_gather_f64(z)
    z_offset = fold_prefix(zs, g)
    total = fold_prefix(zs, G)
    z_bar = total / G
    found = phases.block_boundaries(G, g, z_offset, z_bar)
    b = comm.all_reduce_min_i64(found)
    b[0] = 0
    b[G] = n
    return PlanResult(b, fold_prefix(bws, G), bws, zs, z_bar)


def plan_ucp_distributed(ws, world: int, rank: int) -> np.ndarray:
    """Rank `rank` of `world` GPU processes: the level-1 plan (NCCL)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else None
    comm = TorchComm(device=dev)
    res = plan_ucp_collective(DevicePhases(ws.device), ws.size(), ws.sum_S, world, rank, comm)
    return res.boundaries
