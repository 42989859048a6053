"""Device node_costs_sequential / fill_partition_costs / expected_total_edges,
bit-identical to the reference (cost.cpp:62-77, partition.cpp:205-222,
weights.cpp:155-162): the hand values of test_partition.cpp:55-140 and
test_weights.cpp:191-211, random instances, and every BASELINE.json config
at full size (C4: n = 1e9) for the UCP plans of 2, 4 and 8 GPUs."""
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


def bits(x):
    return np.asarray(x, np.float64).view(np.uint64)


def test_hand_values(api):
    ws = api.make_weight_sequence([2.0, 2.0, 2.0, 2.0])
    assert list(api.fill_partition_costs(api.plan_naive(4, 2), ws)) == pytest.approx([4.5, 2.5], rel=1e-12)
    ws = api.make_weight_sequence([4.0, 3.0, 2.0, 1.0])
    assert list(api.fill_partition_costs(api.plan_rrp(4, 2), ws)) == pytest.approx([4.6, 2.9], rel=1e-12)
    assert list(api.fill_partition_costs(api.plan(ws, "ucp", 2), ws)) == pytest.approx([3.4, 4.1], rel=1e-12)
    assert api.expected_total_edges(ws) == pytest.approx(3.5, rel=1e-12)
    assert api.expected_total_edges(api.make_weight_sequence([2.0] * 4)) == pytest.approx(3.0, rel=1e-12)
    assert api.expected_total_edges(api.make_weight_sequence([7.0])) == 0.0
    assert api.expected_total_edges(api.make_weight_sequence([0.0, 0.0])) == 0.0
    assert list(api.node_costs_sequential(api.make_weight_sequence([0.0, 0.0]))) == [1.0, 1.0]


def test_random_instances_bit_exact(api, ref):
    rng = np.random.default_rng(0xA16)
    for t in range(10):
        n = int(rng.integers(1, 300_000))
        w = np.sort(rng.pareto(1.2, n) * rng.choice([1e-3, 1.0, 1e4]))[::-1].copy()
        if t % 3 == 0:
            w[n // 3:] = 0.0
        ws = api.make_weight_sequence(w)
        rws = ref.weight_sequence(w)
        np.testing.assert_array_equal(bits(api.node_costs_sequential(ws)), bits(ref.node_costs_sequential(rws)))
        assert bits(api.expected_total_edges(ws)) == bits(ref.expected_total_edges(rws))
        for P in (1, 2, 3, 8, 64):
            for scheme in ("naive", "ucp", "rrp"):
                p = api.plan(ws, scheme, P)
                got = api.fill_partition_costs(p, ws)
                exp = ref.fill_partition_costs(rws, scheme, P, p.boundaries)
                np.testing.assert_array_equal(bits(got), bits(exp), err_msg=f"{t} {scheme} {P}")


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_baseline_configs_bit_exact(api, ref, name):
    import inputs
    w = inputs.make(name)
    ws = api.make_weight_sequence(w)
    rws = ref.weight_sequence(w)
    assert bits(api.expected_total_edges(ws)) == bits(ref.expected_total_edges(rws))
    if w.size <= 100_000_000:
        np.testing.assert_array_equal(bits(api.node_costs_sequential(ws)), bits(ref.node_costs_sequential(rws)))
    for G in (2, 4, 8):
        p = api.plan(ws, "ucp", G)
        got = api.fill_partition_costs(p, ws)
        exp = ref.fill_partition_costs(rws, "ucp", G, p.boundaries)
        np.testing.assert_array_equal(bits(got), bits(exp), err_msg=f"{name} G={G}")
        # the planned-cost imbalance the bench reports beside the per-GPU times
        assert got.max() / got.mean() < 1.05
