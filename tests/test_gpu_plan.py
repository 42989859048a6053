"""GPU parity of the level-1 UCP partitioner: boundaries AND the C_u bit
patterns must equal plan_ucp_oracle's (partition.cpp:159-203)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1406_1215_b200 import api as _api
    return _api


def test_plans_match_golden(api):
    plans = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for name, entry in plans.items():
        ws = api.make_weight_sequence(np.array(entry["w"]))
        for key, b in entry.items():
            if key == "w":
                continue
            P = int(key[1:])
            assert list(api.plan_ucp(ws, P)) == b, (name, P)


def test_cost_bit_patterns_match_golden(api):
    g = np.load(os.path.join(GOLDEN, "costs_pl1e5.npz"))
    ws = api.make_weight_sequence(g["w"])
    for P in (1, 2, 4, 8):
        b, cum = api.plan_ucp(ws, P, with_costs=True)
        np.testing.assert_array_equal(cum.view(np.uint64), g[f"cum_P{P}"])
        np.testing.assert_array_equal(b, g[f"plan_P{P}"])


def test_hand_examples_and_contract(api):
    ws = api.make_weight_sequence([4.0, 3.0, 2.0, 1.0])
    assert list(api.plan_ucp(ws, 2)) == [0, 1, 4]          # test_partition.cpp:134-144
    b, cum = api.plan_ucp(ws, 1, with_costs=True)
    assert cum == pytest.approx([3.4, 5.3, 6.5, 7.5], rel=1e-12)  # test_cost.cpp:75-82
    ws3 = api.make_weight_sequence([3.0, 2.0, 1.0])
    assert list(api.plan_ucp(ws3, 1)) == [0, 3]
    for P in (3, 7):
        b = api.plan_ucp(ws3, P)
        assert b[0] == 0 and b[-1] == 3 and np.all(np.diff(b) >= 0)
    with pytest.raises(api.error, match="P must be >= 1"):
        api.plan_ucp(ws, 0)
    empty = api.make_weight_sequence(np.zeros(0))
    assert list(api.plan_ucp(empty, 3)) == [0, 0, 0, 0]
    zeros = api.make_weight_sequence([2.0, 0.0, 0.0, 0.0])
    b, cum = api.plan_ucp(zeros, 1, with_costs=True)


def test_random_plans_vs_oracle(api, port):
    rng = np.random.default_rng(77)
    for t in range(12):
        n = int(rng.integers(1, 200_000))
        scale = rng.choice([1e-3, 1.0, 1e3, 1e6])
        w = np.sort(rng.pareto(1.5, n) * scale)[::-1].copy()
        if t % 3 == 0:
            w[n // 2:] = 0.0
        ws = api.make_weight_sequence(w)
        for P in (1, 2, 3, 4, 8, 16, 64):
            b_ref, cum_ref, _, _ = port.plan_ucp(w, ws.sum_S, P, with_costs=True)
            b, cum = api.plan_ucp(ws, P, with_costs=True)
            np.testing.assert_array_equal(b, b_ref, err_msg=f"trial {t} P {P}")
            np.testing.assert_array_equal(cum.view(np.uint64), cum_ref.view(np.uint64),
                                          err_msg=f"trial {t} P {P}")


def test_c1_plans_match_reference(api):
    s = json.load(open(os.path.join(GOLDEN, "scalars.json")))["c1_continuous"]
    import inputs as workloads
    w = workloads.powerlaw(1_000_000, 2.5, 10.0, 1000.0, 1)
    ws = api.make_weight_sequence(w)
    for P in (2, 4, 8):
        assert list(api.plan_ucp(ws, P)) == s[f"plan_P{P}"]


def test_large_fold_many_binades(api, port):
    # a 20M-element fold crossing many binades, spine + emit on thousands of tiles
    import inputs as workloads
    w = workloads.make("c3", 20_000_000)
    ws = api.make_weight_sequence(w)
    for P in (1, 8):
        b_ref, cum_ref, _, _ = port.plan_ucp(w, ws.sum_S, P, with_costs=True)
        b, cum = api.plan_ucp(ws, P, with_costs=True)
        np.testing.assert_array_equal(b, b_ref)
        np.testing.assert_array_equal(cum.view(np.uint64), cum_ref.view(np.uint64))


def test_distributed_phases_single_process(api, port):
    """The per-rank phases composed on one GPU equal the single-call plan."""
    from paper_1406_1215_b200 import plan
    w = port.synth_powerlaw(300_000, 2.1, 2.0, 1e4, 5)
    ws = api.make_weight_sequence(w)
    for G in (2, 3, 8):
        ph = plan.DevicePhases(ws.device)
        bws = [ph.block_weight(G, g) for g in range(G)]
        zs = [ph.block_costs(G, g, plan.fold_prefix(bws, g), ws.sum_S) for g in range(G)]
        zbar = plan.fold_prefix(zs, G) / G
        found = np.min([ph.block_boundaries(G, g, plan.fold_prefix(zs, g), zbar)
                        for g in range(G)], axis=0)
        found[0], found[G] = 0, len(w)
        np.testing.assert_array_equal(found, port.plan_ucp(w, ws.sum_S, G))
