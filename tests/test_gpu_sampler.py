"""GPU parity tests of the reference-stream sampler against the oracle and the
golden vectors of the real reference (bit-exact: integer edge lists)."""
import json
import os

import numpy as np
import pytest

import stats

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1406_1215_b200 import api as _api
    return _api


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def test_blocked_sum_bit_exact(api, port):
    meta = json.load(open(os.path.join(GOLDEN, "meta.json")))
    for name in meta:
        g = load(f"edges_{name}.npz")
        assert api.blocked_sum(g["w"]) == float(g["S"][0]), name
    rng = np.random.default_rng(3)
    for n in (1, 4095, 4096, 4097, 100_000, 1_234_567):
        x = rng.uniform(0, 1e3, n) * rng.choice([1e-6, 1.0, 1e6], n)
        assert api.blocked_sum(x) == port.blocked_sum(x), n
    s = json.load(open(os.path.join(GOLDEN, "scalars.json")))
    S = api.blocked_sum(np.full(10_000_000, 50.0))
    assert np.array([S]).view(np.uint64)[0] == s["c2_S_bits"]


def test_serial_cl_matches_golden(api):
    meta = json.load(open(os.path.join(GOLDEN, "meta.json")))
    for name, m in meta.items():
        g = load(f"edges_{name}.npz")
        ws = api.make_weight_sequence(g["w"])
        assert ws.sum_S == float(g["S"][0])
        for seed in m["seeds"]:
            edges, flagged = api.serial_cl(ws, seed, return_flagged=True)
            assert flagged == 0
            np.testing.assert_array_equal(edges, g[f"edges_{seed}"], err_msg=f"{name}/{seed}")
        if "range_lo_hi" in g:
            lo, hi = (int(x) for x in g["range_lo_hi"])
            np.testing.assert_array_equal(
                api.create_edges_range(ws, ws.sum_S, lo, hi, m["seeds"][0]), g["edges_range"])
            np.testing.assert_array_equal(
                api.create_edges(ws, ws.sum_S, g["list_sources"], m["seeds"][0]), g["edges_list"])


def test_contract_errors(api):
    ws = api.make_weight_sequence([2.0, 2.0, 2.0, 2.0])
    with pytest.raises(api.error, match="bad node range"):
        api.create_edges_range(ws, ws.sum_S, 0, 5, 1)
    with pytest.raises(api.error, match="bad node range"):
        api.create_edges_range(ws, ws.sum_S, 3, 2, 1)
    with pytest.raises(api.error, match="out of range"):
        api.create_edges(ws, ws.sum_S, [99], 1)
    with pytest.raises(api.error, match="unsorted at position 2"):
        api.make_weight_sequence([3.0, 2.0, 2.5])
    # last node has no destinations (test_edge_skip.cpp:86-90)
    assert len(api.create_edges(ws, ws.sum_S, [3], 1)) == 0
    one = api.make_weight_sequence([5.0])
    assert len(api.serial_cl(one, 3)) == 0
    empty = api.make_weight_sequence(np.zeros(0))
    assert len(api.serial_cl(empty, 3)) == 0


def test_random_instances_vs_oracle(api, port):
    rng = np.random.default_rng(11)
    for t in range(20):
        n = int(rng.integers(2, 3000))
        w = np.sort(rng.uniform(0.0, rng.choice([1.0, 10.0, 100.0]), n))[::-1].copy()
        if t % 5 == 0:
            w[: max(1, n // 50)] *= 50.0  # saturated head: p clamps at 1
            w = np.sort(w)[::-1].copy()
        if t % 7 == 0:
            w[-n // 3:] = 0.0  # zero-weight tail
        ws = api.make_weight_sequence(w)
        seed = int(rng.integers(0, 2**64, dtype=np.uint64))
        got, flagged = api.serial_cl(ws, seed, return_flagged=True)
        exp, cnt, _, _ = port.create_edges_range(w, ws.sum_S, 0, n, seed)
        assert flagged == 0
        np.testing.assert_array_equal(got, exp, err_msg=f"trial {t}")
        counts = api.edge_counts(ws, ws.sum_S, 0, n, seed)
        np.testing.assert_array_equal(counts, port.edge_counts(w, ws.sum_S, 0, n, seed))


def test_c1_continuous_materialised_and_streamed(api, port):
    s = json.load(open(os.path.join(GOLDEN, "scalars.json")))["c1_continuous"]
    w = port.synth_powerlaw(1_000_000, 2.5, 10.0, 1000.0, 1)
    ws = api.make_weight_sequence(w)
    assert np.array([ws.sum_S]).view(np.uint64)[0] == s["S_bits"]
    edges, flagged = api.serial_cl(ws, 7, return_flagged=True)
    assert flagged == 0
    assert len(edges) == s["edges"]
    exp, _, cks, deg = port.create_edges_range(w, ws.sum_S, 0, w.size, 7, degree=True)
    np.testing.assert_array_equal(edges, exp)
    res = api.stream_range(ws, ws.sum_S, 0, w.size, 7, track_shift=0)
    assert res.count == s["edges"]
    assert res.checksum == s["checksum"] == cks
    np.testing.assert_array_equal(res.degree.astype(np.int64), deg)
    res4 = api.stream_range(ws, ws.sum_S, 0, w.size, 7, track_shift=4)
    np.testing.assert_array_equal(res4.degree.astype(np.int64), deg[::16])


def test_device_output_buffer(api, port):
    import torch
    w = port.synth_powerlaw(50_000, 2.5, 2.0, 200.0, 3)
    ws = api.make_weight_sequence(w)
    exp, cnt, _, _ = port.create_edges_range(w, ws.sum_S, 100, 40_000, 9)
    out = torch.empty((cnt + 10, 2), dtype=torch.int32, device="cuda")
    got = api.create_edges_range(ws, ws.sum_S, 100, 40_000, 9, out=out)
    np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), exp)
    small = torch.empty((cnt // 2, 2), dtype=torch.int32, device="cuda")
    with pytest.raises(api.error, match="exceed capacity"):
        api.create_edges_range(ws, ws.sum_S, 100, 40_000, 9, out=small)


def test_ring_emission_matches_checksum(api, port):
    import torch
    w = port.synth_powerlaw(200_000, 2.5, 5.0, 500.0, 4)
    ws = api.make_weight_sequence(w)
    _, cnt, cks, _ = port.create_edges_range(w, ws.sum_S, 0, w.size, 5, materialise=False)
    # per-warp reservations are 2048 slots: size the ring so nothing wraps
    cap = 1 << 25
    assert cnt + 5000 * 2048 < cap
    ring = torch.zeros((cap, 2), dtype=torch.int32, device="cuda")
    res = api.stream_range(ws, ws.sum_S, 0, w.size, 5, ring=ring)
    assert res.count == cnt and res.checksum == cks
    # every edge landed in the ring exactly once (reservation tails stay zero)
    r = ring.cpu().numpy().view(np.uint32).astype(np.uint64)
    nz = r[(r[:, 0] != 0) | (r[:, 1] != 0)]
    assert len(nz) == cnt
    assert stats.checksum(nz) == cks


def test_fast_math_identical_to_reference_expressions(api, port):
    """The guarded fast FP64 path (table log, series log1p, certified
    divisions) must reproduce the reference expressions bit for bit."""
    rng = np.random.default_rng(2025)
    cases = [port.synth_powerlaw(300_000, 2.5, 10.0, 1000.0, 1),      # C1 shape
             np.full(200_000, 50.0),                                   # C2 shape
             port.synth_powerlaw(200_000, 2.1, 2.0, 1e5, 2),           # saturated head
             np.sort(rng.uniform(1e-3, 1.0, 100_000))[::-1].copy(),    # p ~ 1e-8 .. 1e-5
             np.sort(rng.pareto(0.8, 50_000) + 1e-6)[::-1].copy()]     # extreme range
    for i, w in enumerate(cases):
        ws = api.make_weight_sequence(w)
        seed = 1000 + i
        ws.device.set_fast_math(True)
        fast, f1 = api.serial_cl(ws, seed, return_flagged=True)
        ws.device.set_fast_math(False)
        slow, f2 = api.serial_cl(ws, seed, return_flagged=True)
        np.testing.assert_array_equal(fast, slow, err_msg=f"case {i}")
        assert f1 == f2
        if i < 4:  # the extreme-range case legitimately has ratios ~1e12 (2^-47 band)
            assert f1 == 0
        ws.device.set_fast_math(True)
    # and against the oracle on the heaviest case
    w = cases[2]
    ws = api.make_weight_sequence(w)
    exp, _, _, _ = port.create_edges_range(w, ws.sum_S, 0, w.size, 1002)
    np.testing.assert_array_equal(api.serial_cl(ws, 1002), exp)


def test_heavy_phase_is_schedule_only(api, port):
    """The reference stream walks its heaviest chains one per warp (every lane
    on the same chain, lane 0 emitting) before the per-lane phase.  That is a
    schedule: edges, streamed fold, tracked degrees and flags must not change,
    on a partial range as well (the heavy prefix is cut by the range)."""
    cases = [(port.synth_powerlaw(300_000, 2.5, 10.0, 1000.0, 1), 11),   # C1 shape: w >= 256 is heavy
             (port.synth_powerlaw(200_000, 2.1, 2.0, 1e5, 2), 12),       # saturated heavy head (p = 1 prefix)
             (np.full(100_000, 50.0), 13)]                               # no heavy slot at all
    for w, seed in cases:
        ws = api.make_weight_sequence(w)
        n = w.size
        out = {}
        for heavy in (True, False):
            ws.device.set_kernel_shape(-1, heavy_phase=heavy)
            e, nf = api.serial_cl(ws, seed, return_flagged=True)
            lo, hi = 100, n // 3
            part = api.create_edges_range(ws, ws.sum_S, lo, hi, seed)
            st = api.stream_range(ws, ws.sum_S, 0, n, seed, track_shift=2)
            out[heavy] = (e, nf, part, st.count, st.checksum, st.degree.copy())
        ws.device.set_kernel_shape(-1)
        a, b = out[True], out[False]
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[2], b[2])
        assert a[1] == b[1] and a[3] == b[3] and a[4] == b[4]
        np.testing.assert_array_equal(a[5], b[5])
        assert a[3] == len(a[0])
        if seed == 12:  # and against the oracle where the heavy head is saturated
            exp, _, _, _ = port.create_edges_range(w, ws.sum_S, 0, n, seed)
            np.testing.assert_array_equal(a[0], exp)


@pytest.mark.parametrize("env", [
    {"CLGEN_REF_SLOT_SIGMA": "0", "CLGEN_REF_SLOT_CONST": "0"},   # most slots spill
    {"CLGEN_REF_SLOT_SIGMA": "1", "CLGEN_REF_SLOT_CONST": "1"},   # some slots spill
    {"CLGEN_REF_1PASS": "0"},                                      # two-pass path
])
def test_materialise_paths_identical(api, port, env, monkeypatch):
    """Single-pass materialisation (scratch runs + compaction + spill re-walk)
    and the two-pass path produce the reference's edge list exactly."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    dev = api.Device(0)
    rng = np.random.default_rng(21)
    for t in range(6):
        n = int(rng.integers(1000, 60_000))
        w = port.synth_powerlaw(n, 2.2 + 0.1 * t, 1.0, 300.0, t)
        ws = api.make_weight_sequence(w, device=dev)
        lo, hi = int(rng.integers(0, n // 4)), int(rng.integers(n // 2, n + 1))
        exp, cnt, _, _ = port.create_edges_range(w, ws.sum_S, lo, hi, 100 + t)
        np.testing.assert_array_equal(api.create_edges_range(ws, ws.sum_S, lo, hi, 100 + t), exp)
        out = torch.empty((cnt, 2), dtype=torch.int32, device="cuda")
        got = api.create_edges_range(ws, ws.sum_S, lo, hi, 100 + t, out=out)
        np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), exp)
        src = np.unique(rng.integers(0, n, 500)).astype(np.int64)
        exp_l, _, _ = port.create_edges(w, ws.sum_S, src, 5 + t)
        np.testing.assert_array_equal(api.create_edges(ws, ws.sum_S, src, 5 + t), exp_l)


@pytest.mark.parametrize("runs", ["1", "0"])
def test_run_table_bit_exact(api, port, runs, monkeypatch):
    """Repeated weights (discrete, constant, short and tile-crossing runs):
    with and without the run-length table the edges equal the oracle's."""
    monkeypatch.setenv("CLGEN_RUN_TABLE", runs)
    dev = api.Device(0)
    rng = np.random.default_rng(33)
    cases = [np.full(20_000, 7.0),
             np.sort(rng.integers(1, 40, 50_000).astype(np.float64))[::-1].copy(),
             np.sort(np.repeat(rng.uniform(1, 300, 700), rng.integers(1, 6000, 700)))[::-1].copy(),
             np.concatenate([np.full(5000, 900.0), np.full(3, 500.0), np.full(4096 * 3 + 5, 2.0),
                             np.zeros(100)])]
    for t, w in enumerate(cases):
        ws = api.make_weight_sequence(w, device=dev)
        exp, cnt, cks, _ = port.create_edges_range(w, ws.sum_S, 0, w.size, 40 + t)
        np.testing.assert_array_equal(api.create_edges_range(ws, ws.sum_S, 0, w.size, 40 + t), exp,
                                      err_msg=f"case {t}")
        res = api.stream_range(ws, ws.sum_S, 0, w.size, 40 + t)
        assert (res.count, res.checksum) == (cnt, cks)


def test_prefetch_weights_is_plain_ingestion(api, port):
    """clgen_dev_prefetch_weights only moves the host->device copy of the next
    weight array off the critical path: generation from the current weights is
    undisturbed while the copy is in flight, the matching set_weights takes the
    copy (same edges as a plain set_weights), a non-matching one ignores it,
    and the contract checks still run on prefetched data."""
    import torch
    w1 = port.synth_powerlaw(300_000, 2.5, 10.0, 1000.0, 1)
    w2 = port.synth_powerlaw(250_000, 2.1, 2.0, 1e4, 2)
    p1 = torch.from_numpy(w1).pin_memory()
    p2 = torch.from_numpy(w2).pin_memory()
    exp1, _, _, _ = port.create_edges_range(w1, port.blocked_sum(w1), 0, w1.size, 5)
    exp2, _, _, _ = port.create_edges_range(w2, port.blocked_sum(w2), 0, w2.size, 5)

    dev = api.Device(0)

    def edges(w_host):
        ws = api.WeightSequence(w_host, dev.blocked_sum(), None, dev)
        return api.serial_cl(ws, 5)

    dev.set_weights(p1)
    dev.prefetch_weights(p2)                       # in flight while w1 generates
    np.testing.assert_array_equal(edges(w1), exp1)
    dev.set_weights(p2)                            # takes the prefetched copy
    np.testing.assert_array_equal(edges(w2), exp2)
    dev.prefetch_weights(p1)
    dev.set_weights(p2)                            # not the prefetched array: plain copy
    np.testing.assert_array_equal(edges(w2), exp2)
    for _ in range(3):                             # steady state: both buffers cycle
        dev.prefetch_weights(p1)
        dev.set_weights(p1)
        np.testing.assert_array_equal(edges(w1), exp1)
        dev.prefetch_weights(p2)
        dev.set_weights(p2)
        np.testing.assert_array_equal(edges(w2), exp2)
    bad = torch.from_numpy(w1[::-1].copy()).pin_memory()
    dev.prefetch_weights(bad)
    with pytest.raises(api.error, match="weights unsorted"):
        dev.set_weights(bad)
    dev.close()
