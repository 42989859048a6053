"""The counter stream's law on the GPU (SURVEY.md §8(d) gate 3).

* Per-pair frequencies: the reference's own criterion, acceptance.cpp:80-124
  (20 random admissible sequences, n <= 32, weights U(0.2, 2.5), 1e5 trials,
  every pair within 5 sigma of p = min(w_u w_v / S, 1)), ported onto one
  batched launch per sequence (clgen_dev_pair_trials: trial t is exactly the
  generator run with seed base + t).  Three more instance families exercise
  the paths the acceptance weights barely touch: every pair far below
  p = 1/16 (long geometric gaps, many empty chunks), more than 32 weight
  classes (hundreds of class-pair blocks, chunk restarts), and clamped
  pairs / zero weights (dense blocks, exact 0 and 1 frequencies).
* Degree chi^2 at the BASELINE.json sizes with the DEFAULT parameters (class
  automatic class width and chunk size) — the configurations the
  bench reports: (chi^2 - k) / sqrt(2k) <= 5 over the tracked nodes with
  exact FP64 E_i = sum_v min(w_i w_v / S, 1), Var_i = sum_v p (1 - p)
  (acceptance.cpp:113,271 use 4-5 sigma), and the total edge count within
  4 sigma of sum_{u<v} p with the exact Bernoulli variance
  (acceptance.cpp:64-76,268-271).
"""
import numpy as np
import pytest

import stats

pytestmark = pytest.mark.gpu

TRIALS = 100_000
Z_PAIR = 5.0


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1406_1215_b200 import api as _api
    return _api


def pair_z(ws, counts, trials):
    """Worst |f - p| / sigma over pairs u < v; exact frequencies at p in {0, 1}."""
    w = ws.weights
    n = w.size
    S = ws.sum_S
    u, v = np.triu_indices(n, 1)
    p = np.minimum((w[u] * w[v]) / S, 1.0)
    f = counts[u, v] / trials
    lower = np.tril(counts).sum()
    assert lower == 0, "an edge with u >= v"
    sure = (p == 0.0) | (p == 1.0)
    assert np.array_equal(f[sure], p[sure]), "p = 0 / p = 1 pairs must be exact"
    sig = np.sqrt(p * (1 - p) / trials) + 1e-15
    return float(np.max(np.abs(f - p) / sig)), int(u.size)


def random_admissible(rng, n, lo, hi):
    """acceptance.cpp:40-48: U(lo, hi) weights, sorted descending, redrawn
    until admissible (max w^2 < S, weights.cpp:151)."""
    while True:
        w = np.sort(rng.uniform(lo, hi, n))[::-1].copy()
        if w[0] * w[0] < w.sum():
            return w


def test_acceptance_criterion_1_pair_law(api):
    rng = np.random.default_rng(0xC1)
    worst, pairs = 0.0, 0
    for s in range(20):
        n = 4 + int(rng.integers(0, 29))  # up to 32
        w = random_admissible(rng, n, 0.2, 2.5)
        ws = api.make_weight_sequence(w)
        base = int(rng.integers(0, 2**62))
        counts = api.pair_trials(ws, ws.sum_S, base, TRIALS)
        z, k = pair_z(ws, counts, TRIALS)
        worst, pairs = max(worst, z), pairs + k
        assert z < Z_PAIR, (s, n, z)
    assert pairs > 1000


def test_pair_law_small_p(api):
    """Every pair below p = 1/16: sparse blocks with long geometric gaps."""
    rng = np.random.default_rng(0x5A)
    for s in range(6):
        n = 24 + int(rng.integers(0, 9))
        w = random_admissible(rng, n, 0.2, 2.5)
        w = np.concatenate([w, np.full(160, 0.5)])  # light mass that keeps every p small
        w = np.sort(w)[::-1].copy()
        ws = api.make_weight_sequence(w)
        assert (w[0] * w[1]) / ws.sum_S < 1.0 / 16
        counts = api.pair_trials(ws, ws.sum_S, 7000 + s, TRIALS)
        z, _ = pair_z(ws, counts, TRIALS)
        assert z < Z_PAIR, (s, z)


def test_pair_law_many_classes(api):
    """More than 32 weight classes (hundreds of class-pair blocks)."""
    rng = np.random.default_rng(0x3C)
    for s in range(3):
        n = 96
        w = np.sort(np.exp(rng.uniform(np.log(0.05), np.log(5.0), n)))[::-1].copy()
        ws = api.make_weight_sequence(w)
        counts = api.pair_trials(ws, ws.sum_S, 9100 + s, TRIALS)
        info = ws.device.counter_plan_info()
        assert info["classes"] > 32 and info["blocks"] > 32 * 33 // 2, info
        z, _ = pair_z(ws, counts, TRIALS)
        assert z < Z_PAIR, (s, z)


def test_pair_law_clamped_and_zero(api):
    """Clamped pairs (p = 1, dense blocks), near-clamped pairs and zero weights."""
    cases = [np.array([9.0, 8.0, 7.5, 2.0, 1.0, 0.5, 0.25, 0.0, 0.0]),
             np.array([30.0, 30.0, 29.0, 3.0, 2.0, 2.0, 1.0, 1.0, 0.5, 0.1]),
             np.array([4.0, 3.0, 2.0, 1.5, 1.0, 0.5, 0.0])]
    for i, w in enumerate(cases):
        ws = api.make_weight_sequence(w)
        counts = api.pair_trials(ws, ws.sum_S, 777 + i, TRIALS)
        z, _ = pair_z(ws, counts, TRIALS)
        assert z < Z_PAIR, (i, z)
    assert ws.device.counter_plan_info()["dense_blocks"] >= 1


def test_pair_trials_equal_single_runs(api):
    """Trial t of the batched launch is exactly the generator with seed base + t."""
    w = random_admissible(np.random.default_rng(5), 30, 0.2, 2.5)
    ws = api.make_weight_sequence(w)
    base = 123456789
    counts = api.pair_trials(ws, ws.sum_S, base, 40)
    acc = np.zeros_like(counts)
    for t in range(40):
        e = api.generate_range(ws, ws.sum_S, 0, w.size, base + t)
        np.add.at(acc, (e[:, 0], e[:, 1]), 1)
    np.testing.assert_array_equal(counts, acc)


def _chi2_gate(api, ws, w, seed, track_shift, total_z=True):
    res = api.stream_range(ws, ws.sum_S, 0, w.size, seed, mode="counter", track_shift=track_shift)
    nodes = np.arange(0, w.size, 1 << track_shift, dtype=np.int64)
    E, V = stats.expected_degrees(w, ws.sum_S, nodes)
    z, k = stats.chi2_z(res.degree[: nodes.size].astype(np.float64), E, V)
    zt = stats.total_edge_z(res.count, w, ws.sum_S) if total_z else None
    return z, k, zt, res


@pytest.mark.parametrize("name,shift", [("c3", 0), ("c5", 0)])
def test_degree_chi2_full_size_default_params(api, name, shift):
    import inputs
    w = inputs.make(name)
    ws = api.make_weight_sequence(w)
    z, k, zt, res = _chi2_gate(api, ws, w, 2024, shift)
    info = ws.device.counter_plan_info()
    assert info["class_eps"] <= 1.0 / 32, info  # automatic width (1/128, doubled at most twice)
    assert k > 0.9 * w.size
    assert abs(z) <= 5.0, (name, z, k)
    assert abs(zt) <= 4.0, (name, zt)


def test_degree_chi2_c4_full_size(api):
    """C4 at n = 1e9 (the headline workload, bench defaults: track_shift 6,
    1.56e7 tracked nodes; ~2.5e11 edges)."""
    import inputs
    w = inputs.make("c4")
    ws = api.make_weight_sequence(w)
    z, k, _, res = _chi2_gate(api, ws, w, 7, 6, total_z=False)
    assert k > 1.5e7
    assert abs(z) <= 5.0, (z, k)
    # admissible (w0^2 < S): no clamp, so the closed forms of
    # expected_total_edges (weights.cpp:155-162) and of the exact Bernoulli
    # variance (acceptance.cpp:64-76) hold
    S = ws.sum_S
    assert w[0] * w[0] < S
    s2 = float(np.dot(w, w))
    s4 = float(np.dot(w * w, w * w))
    m = (S * S - s2) / (2 * S)
    var = m - (s2 * s2 - s4) / (2 * S * S)
    zt = (res.count - m) / np.sqrt(var)
    assert abs(zt) <= 4.0, zt
