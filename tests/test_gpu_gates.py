"""Full-size deterministic gates (SURVEY.md §8(d) gates 1-2) on the GPU, each
against the UNMODIFIED reference (oracle/_ref) run on the same inputs:

* the level-1 UCP plan of every BASELINE.json config C2-C5 for G in {2,4,8}:
  boundaries equal to plan_ucp_oracle(ws, G) (partition.cpp:159-203) and
  every C_u bit pattern equal to the reference's finalized block profiles
  (cost.cpp:24-51), plus S's bits (weights.cpp:21-30);
* the full C2 edge array (~2.5e8 edges) byte-equal to serial_cl
  (edge_skip.cpp:68-70), the reference run as parallel source ranges;
* reference-stream edges of sampled C3 and C5 sources (heads with the
  longest chains, a random spread, the tail) bit-identical to create_edges
  (edge_skip.cpp:50-58), with no flagged (libm-ambiguous) source.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1406_1215_b200 import api as _api
    return _api


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_size_plans_and_cost_bits_match_reference(api, ref, name):
    import inputs
    w = inputs.make(name)
    ws = api.make_weight_sequence(w)
    rws = ref.weight_sequence(w)
    assert np.array([ws.sum_S]).view(np.uint64)[0] == np.array([rws.sum_S]).view(np.uint64)[0]
    for G in (2, 4, 8):
        b_ref = ref.plan_ucp_oracle(rws, G)
        b, cum = api.plan_ucp(ws, G, with_costs=True)
        np.testing.assert_array_equal(b, b_ref, err_msg=f"{name} G={G}")
        cum_ref, _, _ = ref.global_cum_costs(rws, G)
        bad = np.flatnonzero(cum.view(np.uint64) != cum_ref.view(np.uint64))
        assert bad.size == 0, f"{name} G={G}: {bad.size} C_u bit patterns differ (first {bad[:5]})"
        del cum, cum_ref


def test_c2_full_edge_array_byte_equal(api, ref):
    import inputs
    w = inputs.make("c2")
    n = w.size
    ws = api.make_weight_sequence(w)
    got, flagged = api.serial_cl(ws, 7, return_flagged=True)
    assert flagged == 0
    rws = ref.weight_sequence(w)
    k = 4 * (os.cpu_count() or 8)
    cuts = np.linspace(0, n, k + 1).astype(np.int64)

    def part(i):
        return ref.create_edges_range(rws, rws.sum_S, int(cuts[i]), int(cuts[i + 1]), 7)[0]

    with ThreadPoolExecutor(os.cpu_count() or 8) as ex:
        exp = np.concatenate(list(ex.map(part, range(k))))
    assert got.shape == exp.shape and got.shape[0] > 2.4e8
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("name,nsample", [("c3", 4000), ("c5", 4000)])
def test_reference_stream_sampled_sources_bit_exact(api, ref, name, nsample):
    import inputs
    w = inputs.make(name)
    n = w.size
    ws = api.make_weight_sequence(w)
    rws = ref.weight_sequence(w)
    rng = np.random.default_rng(0x5E)
    src = np.unique(np.concatenate([np.arange(0, 64), rng.integers(0, n, nsample),
                                    np.arange(n - 64, n)])).astype(np.int64)
    got, flagged = api.create_edges(ws, ws.sum_S, src, 7, return_flagged=True)
    assert flagged == 0, f"{name}: {flagged} sources in the libm-ambiguity band"
    exp, _ = ref.create_edges(rws, rws.sum_S, src, 7)
    np.testing.assert_array_equal(got, exp)
