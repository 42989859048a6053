"""CPU tests: pin the C restatement (oracle/clgen_oracle.c) against the
reference's own known answers and against golden vectors produced by the
unmodified reference (tests/golden/make_golden.py)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

import oracle


def load(name):
    return np.load(os.path.join(GOLDEN, name))


# ---- known answers copied from the reference's tests ---------------------

def test_skip_length_hand_values(port):
    # test_edge_skip.cpp:42-64
    assert port.skip_length(1.0, 0.9) == 0
    assert port.skip_length(1.0, 1e-12) == 0
    assert port.skip_length(0.5, 0.25) == 2
    assert port.skip_length(0.5, 0.6) == 0
    for p, r in [(0.0, 0.5), (-0.1, 0.5), (1.5, 0.5), (0.5, 0.0), (0.5, 1.0)]:
        with pytest.raises(oracle.OracleError):
            port.skip_length(p, r)
    assert port.skip_length(1e-300, 0.5) == np.iinfo(np.int64).max


def test_node_cost_hand_values(port):
    # test_cost.cpp:49-60
    assert port.node_cost(4.0, 0.0, 10.0) == pytest.approx(3.4, rel=1e-12)
    assert port.node_cost(2.0, 2.0, 8.0) == pytest.approx(2.0, rel=1e-12)
    assert port.node_cost(1.0, 9.0, 10.0) == 1.0
    assert port.node_cost(1.0, 9.5, 10.0) == 1.0
    with pytest.raises(oracle.OracleError):
        port.node_cost(1.0, 0.0, 0.0)


def test_block_bounds_ceil_first(port):
    # test_cost.cpp:62-73
    assert port.block_bounds(4, 2, 0) == (0, 2)
    assert port.block_bounds(4, 2, 1) == (2, 4)
    assert port.block_bounds(5, 2, 0) == (0, 3)
    assert port.block_bounds(5, 2, 1) == (3, 5)
    assert port.block_bounds(3, 8, 2) == (2, 3)
    assert port.block_bounds(3, 8, 5) == (3, 3)
    with pytest.raises(oracle.OracleError):
        port.block_bounds(4, 0, 0)


def test_block_cumulative_hand_values(port):
    # test_cost.cpp:75-94
    w = np.array([4.0, 3.0, 2.0, 1.0])
    cum, bc = port.block_cumulative(w, 10.0, 0, 1, 0.0)
    assert cum == pytest.approx([3.4, 5.3, 6.5, 7.5], rel=1e-12)
    assert bc == cum[-1]
    cum, bc = port.block_cumulative(w, 10.0, 1, 2, 7.0)
    assert cum == pytest.approx([1.2, 2.2], rel=1e-12)
    z = np.array([2.0, 0.0, 0.0, 0.0])
    cum, _ = port.block_cumulative(z, 2.0, 1, 2, 2.0)
    assert list(cum) == [1.0, 2.0]


def test_partition_of(port):
    # test_cost.cpp:113-120
    assert port.partition_of(3.4, 3.75, 2) == 0
    assert port.partition_of(5.3, 3.75, 2) == 1
    assert port.partition_of(7.5, 3.75, 2) == 1
    assert port.partition_of(0.0, 1.0, 4) == 0
    with pytest.raises(oracle.OracleError):
        port.partition_of(1.0, 0.0, 2)


def test_plan_hand_examples(port):
    # test_partition.cpp:134-160
    w = np.array([4.0, 3.0, 2.0, 1.0])
    assert list(port.plan_ucp(w, 10.0, 2)) == [0, 1, 4]
    w = np.array([3.0, 2.0, 1.0])
    assert list(port.plan_ucp(w, 6.0, 1)) == [0, 3]
    for P in (3, 7):
        b = port.plan_ucp(w, 6.0, P)
        assert b[0] == 0 and b[-1] == 3 and np.all(np.diff(b) >= 0)


def test_dominant_node_has_empty_partitions(port):
    # test_partition.cpp:106-132
    w = np.array([40.0] + [1.0] * 7)
    b = port.plan_ucp(w, port.blocked_sum(w), 4)
    assert np.any(np.diff(b) == 0)


def test_synth_constant_sum():
    # c2: S = 5e8 exactly
    P = oracle.port()
    w = np.full(10_000_000, 50.0)
    assert P.blocked_sum(w) == 5e8


# ---- port vs golden vectors from the real reference ----------------------

def test_port_matches_golden_edges(port):
    meta = json.load(open(os.path.join(GOLDEN, "meta.json")))
    for name, m in meta.items():
        g = load(f"edges_{name}.npz")
        w, S = g["w"], float(g["S"][0])
        assert port.blocked_sum(w) == S
        for seed in m["seeds"]:
            pairs, cnt, _, _ = port.create_edges_range(w, S, 0, w.size, seed)
            np.testing.assert_array_equal(pairs, g[f"edges_{seed}"], err_msg=f"{name} seed {seed}")
        if "range_lo_hi" in g:
            lo, hi = (int(x) for x in g["range_lo_hi"])
            pairs, _, _, _ = port.create_edges_range(w, S, lo, hi, m["seeds"][0])
            np.testing.assert_array_equal(pairs, g["edges_range"])
            pairs, _, _ = port.create_edges(w, S, g["list_sources"], m["seeds"][0])
            np.testing.assert_array_equal(pairs, g["edges_list"])


def test_port_matches_golden_plans(port):
    plans = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for name, entry in plans.items():
        w = np.array(entry["w"])
        S = port.blocked_sum(w)
        for key, b in entry.items():
            if key == "w":
                continue
            P = int(key[1:])
            assert list(port.plan_ucp(w, S, P)) == b, (name, P)


def test_port_matches_golden_costs(port):
    g = load("costs_pl1e5.npz")
    w, S = g["w"], float(g["S"][0])
    for P in (1, 2, 4, 8):
        b, cum, bw, bc = port.plan_ucp(w, S, P, with_costs=True)
        np.testing.assert_array_equal(cum.view(np.uint64), g[f"cum_P{P}"])
        np.testing.assert_array_equal(bw.view(np.uint64), g[f"bw_P{P}"])
        np.testing.assert_array_equal(bc.view(np.uint64), g[f"bc_P{P}"])
        np.testing.assert_array_equal(b, g[f"plan_P{P}"])


def test_port_matches_golden_skip(port):
    s = json.load(open(os.path.join(GOLDEN, "scalars.json")))
    for p, r, d in s["skip"]:
        assert port.skip_length(p, r) == d


@pytest.mark.slow
def test_port_c1_continuous_headline(port):
    s = json.load(open(os.path.join(GOLDEN, "scalars.json")))["c1_continuous"]
    w = port.synth_powerlaw(1_000_000, 2.5, 10.0, 1000.0, 1)
    S = port.blocked_sum(w)
    assert np.array([S]).view(np.uint64)[0] == s["S_bits"]
    _, cnt, cks, _ = port.create_edges_range(w, S, 0, w.size, 7, materialise=False)
    assert cnt == s["edges"] == 13516657
    assert cks == s["checksum"] == 0x7DF0117BC9E92264
    assert list(port.plan_ucp(w, S, 8)) == s["plan_P8"]


# ---- port vs live reference (only where the reference build exists) -------

def test_port_vs_reference_random(port, ref):
    rng = np.random.default_rng(5)
    for t in range(6):
        n = int(rng.integers(2, 400))
        w = np.sort(rng.uniform(0.0, 5.0, n))[::-1].copy()
        ws = ref.weight_sequence(w)
        S = ws.sum_S
        assert port.blocked_sum(w) == S
        seed = int(rng.integers(0, 2**63))
        a, _ = ref.create_edges_range(ws, S, 0, n, seed)
        b, _, _, _ = port.create_edges_range(w, S, 0, n, seed)
        np.testing.assert_array_equal(a, b)
        for P in (2, 5, 16):
            np.testing.assert_array_equal(ref.plan_ucp_oracle(ws, P), port.plan_ucp(w, S, P))


def test_port_synth_matches_reference(port, ref):
    ws = ref.synth_powerlaw(5000, 2.1, 2.0, 1e5, 1)
    np.testing.assert_array_equal(ws.weights, port.synth_powerlaw(5000, 2.1, 2.0, 1e5, 1))
    assert ws.sum_S == port.blocked_sum(ws.weights)


def test_input_synthesis_bit_identical_to_reference(ref):
    """inputs (both bench arms' input preparation, libclgen_inputs.so) draws
    synth_powerlaw's values bit for bit (weights.cpp:103-128; the reference
    stable-sorts them, make_weight_sequence at :32-55) and synth_constant's
    (:130-140) — for the C1/C3/C4/C5 parameter sets at n = 2e5."""
    import inputs
    for n, gamma, lo, hi, seed in ((200_000, 2.5, 10.0, 1000.0, 1), (200_000, 2.1, 2.0, 1e5, 1),
                                   (200_000, 2.5, 1.0, 1000.0, 1), (200_000, 2.0, 1.0, 977.0, 3)):
        got = inputs.powerlaw(n, gamma, lo, hi, seed)
        exp = ref.synth_powerlaw(n, gamma, lo, hi, seed).weights
        assert got.view(np.uint64).tolist() == exp.view(np.uint64).tolist()
    c = ref.synth_constant(1000, 50.0)
    assert np.array_equal(c.weights, np.full(1000, 50.0)) and c.sum_S == 50000.0
