"""Per-rank runtime around the device generator (the generate_on_rank analogue,
/root/reference/proj/core/src/runtime.cpp:46-91): weight distribution to the
ranks, the level-1 UCP plan over the GPUs, and end-to-end measurement helpers
used by bench.py.  One process per GPU; torch.distributed (NCCL) carries the
plan's tiny collectives.
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def comm_device(local: int):
    """Tensor device for collectives: the GPU for NCCL, the host for gloo."""
    import torch
    import torch.distributed as dist
    return torch.device(f"cuda:{local}") if dist.get_backend() == "nccl" else torch.device("cpu")


# inputs.make's synth_powerlaw recipes: gamma, w_min, w_max, synth seed, target mean
DEVICE_RECIPES = {"c3": (2.1, 2.0, 1e5, 1, 0.0), "c4": (2.5, 1.0, 1000.0, 1, 500.0)}


def shared_weights(config: str, n: int | None, world: int, rank: int, local: int) -> np.ndarray:
    """Every rank holds all of w.  Rank 0 synthesises the
    workload's weights (input preparation, ``inputs``) into a host file that
    the other ranks map; nothing but a barrier crosses the process group, so
    the only NCCL traffic of a run stays the plan's scalars."""
    import inputs
    if config in DEVICE_RECIPES and os.environ.get("CLGEN_HOST_SYNTH", "0") != "1":
        # continuous power-law recipes: every rank synthesises the array on its
        # own GPU (clgen_dev_synth_powerlaw: bit-identical to inputs.make, which
        # the CPU reference arm keeps using) and reads it back once
        import torch
        gamma, w_min, w_max, seed, mean = DEVICE_RECIPES[config]
        w_dev, _ = api.synth_powerlaw_device(n or inputs.WORKLOADS[config].n, gamma, w_min, w_max, seed,
                                             api.default_device(local), True, mean)
        w = w_dev.cpu().numpy()
        del w_dev
        torch.cuda.empty_cache()
        return w
    if world == 1:
        return inputs.make(config, n)
    import torch.distributed as dist
    tag = os.environ.get("MASTER_PORT", "0")
    shm = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
    path = os.path.join(shm, f"clgen_w_{config}_{n or 0}_{tag}.f64")
    w = None
    if rank == 0:
        w = inputs.make(config, n)
        w.tofile(path + ".part")
        os.replace(path + ".part", path)
    dist.barrier()
    if rank != 0:
        w = np.fromfile(path, dtype=np.float64)
    dist.barrier()
    if rank == 0:
        os.remove(path)
    return w


def plan(ws: api.WeightSequence, world: int, rank: int) -> np.ndarray:
    """Level-1 UCP boundaries over `world` GPUs, bit-identical to
    plan_ucp_oracle(ws, world) (partition.cpp:159-203)."""
    if world == 1:
        return np.array([0, ws.size()], np.int64)
    from . import plan as _plan
    return _plan.plan_ucp_distributed(ws, world, rank)


def plan_phase_times(dev, n: int, S: float, G: int) -> dict:
    """The level-1 plan's three per-rank device phases for G ranks
    (partition.cpp:115-154: block weight, block_cumulative, boundaries), run
    rank after rank on this one GPU and host-timed (each phase returns a
    scalar, i.e. synchronises).  Max over ranks of the per-rank sum is the
    device time each GPU of a G-GPU run spends planning (the NCCL
    all-gathers / all-reduce between the phases carry 8-byte payloads and
    are not included)."""
    import time
    from .plan import DevicePhases, fold_prefix
    ph = DevicePhases(dev)
    t_bw, t_bc, t_bd, bws, zs = [], [], [], [], []
    for g in range(G):
        t0 = time.perf_counter()
        bws.append(ph.block_weight(G, g))
        t_bw.append((time.perf_counter() - t0) * 1e3)
    for g in range(G):
        t0 = time.perf_counter()
        zs.append(ph.block_costs(G, g, fold_prefix(bws, g), S))
        t_bc.append((time.perf_counter() - t0) * 1e3)
    z_bar = fold_prefix(zs, G) / G
    found = []
    for g in range(G):
        t0 = time.perf_counter()
        found.append(ph.block_boundaries(G, g, fold_prefix(zs, g), z_bar))
        t_bd.append((time.perf_counter() - t0) * 1e3)
    b = np.min(np.stack(found), axis=0)
    b[0], b[G] = 0, n
    per_rank = [a + c + d for a, c, d in zip(t_bw, t_bc, t_bd)]
    # planned cost per GPU (fill_partition_costs, partition.cpp:205-222)
    ws = api.WeightSequence(np.empty(0), S, None, dev)
    planned = api.fill_partition_costs(api.PartitionPlan("ucp", G, n, b), ws)
    return {"G": G, "block_weight_ms": [round(x, 3) for x in t_bw],
            "block_costs_ms": [round(x, 3) for x in t_bc],
            "boundaries_ms": [round(x, 3) for x in t_bd],
            "per_rank_max_ms": round(max(per_rank), 3), "boundaries": b.tolist(),
            "planned_cost_max_over_mean": float(planned.max() / planned.mean())}


def expected_edges(w: np.ndarray, S: float, lo: int, hi: int) -> float:
    """Expected edges of sources [lo,hi) (unclamped, an upper bound of the
    clamped mean) plus a 6-sigma margin: capacity sizing only."""
    if hi <= lo or not S > 0:
        return 0.0
    suffix = S - np.cumsum(w, dtype=np.float64)
    e = float((w[lo:hi] / S * suffix[lo:hi]).sum())
    return e + 6.0 * np.sqrt(max(e, 1.0))


def ncu_traffic(config: str, mode: str):
    """DRAM bytes per sampler launch from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(f"{config}:{mode}")
    except Exception:
        return None


def e2e_measure(args, w_host: np.ndarray, world: int, rank: int, local: int, lo: int, hi: int,
                seed: int, materialise: bool) -> dict:
    """The same metric through the public API with HOST buffers: every step
    copies the weights host->device (pinned), recomputes S and the plan, runs
    the generator and reads the result back (edges for materialised configs,
    count/checksum/tracked degrees for streaming ones)."""
    import torch
    n = int(w_host.size)
    # page-lock the caller's weight array in place (no second 8 GB host copy
    # per rank); fall back to a pinned copy if registration is refused
    w_host = np.ascontiguousarray(w_host)
    cudart = torch.cuda.cudart()
    registered = int(cudart.cudaHostRegister(w_host.ctypes.data, w_host.nbytes, 0)) == 0
    if registered:
        pinned = w_host
    else:
        pinned = torch.empty(n, dtype=torch.float64, pin_memory=True)
        pinned.numpy()[:] = w_host
    dev = api.Device(local)
    stream = dev.torch_stream()
    # ingestion pipelining: every step still copies its weights host->device
    # inside the timed region, but the copy for step k+1 is issued on the
    # context's copy stream while step k generates (double-buffered weights)
    pipelined = os.environ.get("CLGEN_E2E_PIPELINE", "1") != "0"
    ring = None
    host_out = None
    deg_host = None
    if materialise:
        cap = int(expected_edges(w_host, float(np.sum(w_host)), lo, hi) * 1.01 + 1_000_000)
        host_out = torch.empty((cap, 2), dtype=torch.int32, pin_memory=True)
    else:
        ring = torch.empty((1 << args.ring_log2, 2), dtype=torch.int32, device=f"cuda:{local}")
        ntr = (n + (1 << args.track_shift) - 1) >> args.track_shift
        deg_host = torch.zeros(ntr, dtype=torch.int32, pin_memory=True)

    def one():
        dev.set_weights(pinned)                      # H2D (n * 8 bytes), or the copy prefetched last step
        S = dev.blocked_sum()
        ws = api.WeightSequence(w_host, S, None, dev)
        b = plan(ws, world, rank)
        a, z = int(b[rank]), int(b[rank + 1])
        if pipelined:
            dev.prefetch_weights(pinned)             # next step's H2D, under this step's generation
        if materialise:
            e = api.create_edges_range(ws, S, a, z, seed, out=host_out)  # D2H of the edges
            return int(e.shape[0]), int(e.shape[0]) * 8
        r = api.stream_range(ws, S, a, z, seed, mode=args.mode, track_shift=args.track_shift,
                             degree=deg_host.numpy(), ring=ring)     # D2H of tracked degrees
        return r.count, deg_host.numel() * 4 + 16

    one()
    torch.cuda.synchronize()
    total_ms, edges = 0.0, 0
    d2h = 0
    for _ in range(args.steps):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        c, d2h = one()
        ev1.record(stream)
        ev1.synchronize()
        total_ms += ev0.elapsed_time(ev1)
        edges += c
    ms = total_ms / args.steps
    e_step = edges // args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=comm_device(local))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e = torch.tensor([e_step], dtype=torch.int64, device=comm_device(local))
        dist.all_reduce(e)
        ms, e_step = float(t[0]), int(e[0])
    dev.close()
    if registered:
        cudart.cudaHostUnregister(w_host.ctypes.data)
    return {"value": e_step / (ms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": n * 8,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "h2d": "next step's copy overlapped with this step (clgen_dev_prefetch_weights)" if pipelined
            else "serial"}
