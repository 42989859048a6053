"""GPU tests of the §8(f) rows (f2) edge files and (f3) naive/RRP plans:
acceptance.cpp:298-337's determinism & scheme invariance — merged, sorted
edge files byte-identical across {naive, ucp, rrp} x P in {1,2,4,8} — with the
files written by the device writer and compared with the reference's own
write_edges bytes."""
import os

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


def test_scheme_invariance_byte_identical(api, ref, tmp_path):
    rws = ref.synth_powerlaw(3000, 2.5, 2.0, 50.0, 0xDE7)  # acceptance.cpp:299
    ws = api.make_weight_sequence(rws.weights)
    exp, _ = ref.create_edges_range(rws, rws.sum_S, 0, rws.n, 1234)
    ref_path = str(tmp_path / "ref.bin")
    ref.write_edges(exp, ref_path, binary=True)
    ref_bytes = open(ref_path, "rb").read()
    for scheme in ("naive", "ucp", "rrp"):
        for P in (1, 2, 4, 8):
            plan = api.plan(ws, scheme, P)
            parts = [api.generate_partition(ws, plan, i, 1234) for i in range(P)]
            merged = np.concatenate([p for p in parts if len(p)] or [np.zeros((0, 2), np.uint32)])
            key = merged[:, 0].astype(np.int64) * ws.n + merged[:, 1]
            merged = merged[np.argsort(key, kind="stable")]
            path = str(tmp_path / f"{scheme}{P}.bin")
            api.write_edges(merged, path, "binary", device=ws.device)
            assert open(path, "rb").read() == ref_bytes, (scheme, P)


def test_text_and_roundtrip(api, ref, tmp_path):
    rng = np.random.default_rng(3)
    e = np.sort(rng.integers(0, 2**32 - 1, size=(100_003, 2), dtype=np.uint64), axis=1).astype(np.uint32)
    for fmt, binary in (("text", False), ("binary", True)):
        ours, theirs = str(tmp_path / f"o.{fmt}"), str(tmp_path / f"r.{fmt}")
        api.write_edges(e, ours, fmt)
        ref.write_edges(e, theirs, binary=binary)
        assert open(ours, "rb").read() == open(theirs, "rb").read(), fmt
        np.testing.assert_array_equal(api.read_edges(ours), e)
        np.testing.assert_array_equal(ref.read_edges(ours), e)
    empty = str(tmp_path / "empty.bin")
    api.write_edges(np.zeros((0, 2), np.uint32), empty, "binary")
    assert len(api.read_edges(empty)) == 0
    with pytest.raises(api.error, match="cannot open for writing"):
        api.write_edges(e, str(tmp_path / "no" / "such" / "dir.bin"))


def test_device_tensor_input(api, tmp_path):
    import torch
    e = torch.randint(0, 1 << 30, (5000, 2), dtype=torch.int32, device="cuda")
    p = str(tmp_path / "d.bin")
    api.write_edges(e, p)
    np.testing.assert_array_equal(api.read_edges(p), e.cpu().numpy().view(np.uint32))


def test_plan_shapes(api):
    p = api.plan_naive(5, 2)
    assert list(p.boundaries) == [0, 3, 5]          # test_partition.cpp:58
    assert list(api.plan_naive(3, 5).boundaries) == [0, 1, 2, 3, 3, 3]
    r = api.plan_rrp(5, 2)
    assert list(r.partition_nodes(0)) == [0, 2, 4] and list(r.partition_nodes(1)) == [1, 3]
    assert r.partition_size(0) == 3 and r.partition_size(1) == 2
    with pytest.raises(api.error):
        api.plan_naive(4, 0)


def test_fidelity_matches_reference(api, ref):
    """(f1): device degree-fidelity report == analysis.cpp's, bit for bit."""
    for (n, g, lo, hi, s_w, s_g) in [(100_000, 2.5, 50.0, 800.0, 0xF1DF, 0xF1E0),  # acceptance.cpp:276
                                     (200_000, 2.1, 2.0, 1e4, 5, 6)]:
        rws = ref.synth_powerlaw(n, g, lo, hi, s_w)
        ws = api.make_weight_sequence(rws.weights)
        edges = api.serial_cl(ws, s_g)
        ours_deg = api.edge_degrees(ws, edges)
        streamed = api.stream_range(ws, ws.sum_S, 0, n, s_g, track_shift=0)
        np.testing.assert_array_equal(streamed.degree, ours_deg)
        got = api.fidelity(ws, ours_deg, len(edges), 100.0)
        exp = ref.fidelity(rws, edges, 100.0)
        for key in ("mean_expected", "mean_generated", "mean_rel_error", "max_flagged_rel_error",
                    "zero_degree"):
            assert got[key] == exp[key], key
        assert got["bins"] == exp["bins"]
    # constant weights (acceptance.cpp:260-266): mean degree within 2%
    cws = api.make_weight_sequence(np.full(100_000, 50.0))
    r = api.stream_range(cws, cws.sum_S, 0, 100_000, 0xF1DE, track_shift=0)
    rep = api.fidelity(cws, r.degree, r.count)
    assert rep["mean_rel_error"] <= 0.02
