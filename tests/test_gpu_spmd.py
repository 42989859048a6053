"""Multi-rank paths on one GPU (the box this suite runs on has one).

* clgen_spmd_generate — the generate()/run_spmd analogue (runtime.cpp:93-138,
  comm.cpp:204-227): one host thread per rank.  G = 1 exercises the NCCL
  communicator (ncclCommInitAll on the device); G > 1 ranks share the device
  and use the in-process host communicator.  The plan must equal
  plan_ucp_oracle(ws, G) and the union of the ranks' streams must be the
  single-range stream (both random streams).
* The torch.distributed path of bench.py (plan.plan_ucp_collective with the
  DEVICE phases through the C ABI) over gloo, world size 2, both ranks on
  cuda:0, on a C3-shaped input at n = 1e7: boundaries equal to the
  reference's plan_ucp_oracle (partition.cpp:159-203).
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1406_1215_b200 import api as _api
    return _api


@pytest.mark.parametrize("mode", ["counter", "reference"])
def test_spmd_generate_matches_plan_and_single_stream(api, ref, mode):
    import inputs
    w = inputs.make("c3", 2_000_000)
    ws = api.make_weight_sequence(w)
    full = api.stream_range(ws, ws.sum_S, 0, w.size, 5, mode=mode)
    rws = ref.weight_sequence(w)
    for devs in ([0], [0, 0], [0, 0, 0, 0]):
        G = len(devs)
        r = api.spmd_generate(w, devs, 5, mode=mode)
        np.testing.assert_array_equal(r["boundaries"], ref.plan_ucp_oracle(rws, G))
        assert (r["total_edges"], r["checksum"]) == (full.count, full.checksum), devs
        assert int(r["rank_edges"].sum()) == r["total_edges"]
        assert r["S"] == ws.sum_S and r["n_flagged"] == 0
        if G == 1:
            assert r["nccl_version"] > 0  # the NCCL communicator carried the collectives
        else:
            assert r["nccl_version"] == 0


def test_spmd_generate_errors_like_the_reference(api):
    with pytest.raises(api.error, match="weights unsorted"):
        api.spmd_generate(np.array([1.0, 2.0, 3.0]), [0, 0], 1)


def _worker(rank, world, port_no, w, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1406_1215_b200 import api, plan
    dev = api.Device(0)  # both ranks on the one GPU (CLGEN_DEVICE_OVERRIDE in bench.py)
    dev.set_weights(w)
    S = dev.blocked_sum()
    res = plan.plan_ucp_collective(plan.DevicePhases(dev), w.size, S, world, rank, plan.TorchComm())
    out[rank] = (res.boundaries.tolist(), res.reduced_sum, S)
    dev.close()
    dist.destroy_process_group()


def test_torch_distributed_plan_with_device_phases(ref):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    import inputs
    w = inputs.make("c3", 10_000_000)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port_no, w, out), nprocs=world, join=True)
    rws = ref.weight_sequence(w)
    expect = ref.plan_ucp_oracle(rws, world).tolist()
    for r in range(world):
        b, reduced, S = out[r]
        assert b == expect, (r, b, expect)
        assert S == rws.sum_S


def _nccl_worker(rank, world, port_no, w, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda:0"))
    from paper_1406_1215_b200 import api, plan, runtime
    ws = api.make_weight_sequence(w, device=0)
    dist.barrier()
    b = plan.plan_ucp_distributed(ws, world, rank)  # the bench's own call: NCCL tensors on the GPU
    comm = plan.TorchComm(device=runtime.comm_device(0))
    g = comm.all_gather_f64(ws.sum_S)
    m = comm.all_reduce_min_i64(np.array([3, 1, 2], np.int64))
    out[rank] = (b.tolist(), g.tolist(), m.tolist(), dist.get_backend())
    ws.device.close()
    dist.destroy_process_group()


def test_bench_plan_path_over_nccl_single_rank():
    """bench.py --gpus N plans through torch.distributed over NCCL with device
    tensors.  This box has one GPU, so the communicator has one rank: what is
    pinned here is that the NCCL code path itself (process-group init on the
    device, barrier, float64 all_gather_into_tensor, int64 MIN all_reduce on
    GPU tensors) runs and returns the right values."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    import inputs
    w = inputs.make("c3", 1_000_000)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_nccl_worker, args=(1, port_no, w, out), nprocs=1, join=True)
    b, g, m, backend = out[0]
    assert backend == "nccl"
    assert b == [0, w.size]
    assert len(g) == 1 and g[0] > 0.0
    assert m == [3, 1, 2]
