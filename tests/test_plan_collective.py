"""CPU test of the multi-GPU plan orchestration (plan_ucp_collective) with
world_size 2/3 over gloo: the device phases are stood in by the oracle's C
restatement, the collectives are the real torch.distributed ones."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


class OraclePhases:
    """Per-rank phases computed by the oracle (tests only)."""

    def __init__(self, w, S):
        import oracle
        self.p = oracle.port()
        self.w, self.S = w, S

    def block_weight(self, G, g):
        lo, hi = self.p.block_bounds(self.w.size, G, g)
        acc = 0.0
        for x in self.w[lo:hi].tolist():
            acc += x
        return acc

    def block_costs(self, G, g, sigma_start, S):
        self.cum, z = self.p.block_cumulative(self.w, S, g, G, sigma_start)
        self.lo, _ = self.p.block_bounds(self.w.size, G, g)
        return z

    def block_boundaries(self, G, g, z_offset, z_bar):
        found = np.full(G + 1, self.w.size, np.int64)
        prev = self.p.partition_of(z_offset, z_bar, G)
        for i, c in enumerate(self.cum.tolist()):
            cur = self.p.partition_of(c + z_offset, z_bar, G)
            for k in range(prev + 1, cur + 1):
                found[k] = self.lo + i
            prev = cur
        return found


def _worker(rank, world, port_no, w, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1406_1215_b200 import plan
    import oracle
    S = oracle.port().blocked_sum(w)
    res = plan.plan_ucp_collective(OraclePhases(w, S), w.size, S, world, rank, plan.TorchComm())
    out[rank] = (res.boundaries.tolist(), res.reduced_sum)
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_collective_plan_matches_oracle(world, port):
    rng = np.random.default_rng(world)
    w = np.sort(rng.pareto(1.2, 5000) + 0.1)[::-1].copy()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), w, out), nprocs=world, join=True)
    S = port.blocked_sum(w)
    ref = port.plan_ucp(w, S, world).tolist()
    for r in range(world):
        b, reduced = out[r]
        assert b == ref
        # the reduced sum is the reference's rank-ordered all_reduce (runtime.cpp:55-58)
        acc = 0.0
        for g in range(world):
            lo, hi = port.block_bounds(w.size, world, g)
            part = 0.0
            for x in w[lo:hi].tolist():
                part += x
            acc += part
        assert reduced == acc


def test_dominant_node_empty_partitions(port):
    w = np.array([4000.0] + [1.0] * 60)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, free_port(), w, out), nprocs=2, join=True)
    assert out[0][0] == port.plan_ucp(w, port.blocked_sum(w), 2).tolist()
