"""Regenerate the golden fixtures in tests/golden/ from the REAL reference.

Runs the unmodified reference library (oracle/_ref/libclgen_ref.so, compiled
from /root/reference/proj/core/src by oracle/Makefile) on seeded inputs and
stores inputs + outputs as small .npz files.  Only this script and the CPU
tests need /root/reference; the fixtures travel with the repo to the GPU box.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def random_admissible(rng: np.random.Generator, n: int, lo: float, hi: float) -> np.ndarray:
    """Sorted weights with max w^2 < S (the reference tests' random_admissible)."""
    while True:
        w = np.sort(rng.uniform(lo, hi, n))[::-1].copy()
        if w[0] * w[0] < w.sum():
            return w


def main() -> None:
    oracle.build(ref=True)
    R = oracle.ref()
    rng = np.random.default_rng(20241020)
    meta = {}

    # ---- edge sets of small instances (serial_cl, create_edges_range) ----
    cases = {
        "const4": (np.array([2.0, 2.0, 2.0, 2.0]), [7, 8, 9]),
        "dyadic": (np.array([4.0] * 96 + [2.0] * 64), [1, 2]),
        "clamped": (np.array([4.0, 3.0, 2.0]), [0, 1, 2, 3]),
        "zero_tail": (np.array([3.0, 2.0, 1.0, 0.0, 0.0]), [0, 5, 11]),
        "single": (np.array([5.0]), [3]),
        "adm64": (random_admissible(rng, 64, 0.2, 3.0), [424242]),
        "adm200": (random_admissible(rng, 200, 0.2, 3.0), [0, 1, 2]),
        "dominant": (np.array([4000.0] + [1.0] * 63), [5]),
        "pl3000": (R.synth_powerlaw(3000, 2.5, 2.0, 50.0, 0xDE7).weights, [1234]),
        "pl20000": (R.synth_powerlaw(20000, 2.1, 1.0, 2000.0, 99).weights, [7]),
    }
    for name, (w, seeds) in cases.items():
        ws = R.weight_sequence(w)
        store = {"w": w, "S": np.array([ws.sum_S])}
        for seed in seeds:
            pairs, cnt = R.create_edges_range(ws, ws.sum_S, 0, ws.n, seed)
            store[f"edges_{seed}"] = pairs
        # a sub-range and an explicit source list (create_edges order)
        if ws.n >= 8:
            lo, hi = ws.n // 4, ws.n // 2
            pairs, _ = R.create_edges_range(ws, ws.sum_S, lo, hi, seeds[0])
            store["range_lo_hi"] = np.array([lo, hi])
            store["edges_range"] = pairs
            src = rng.permutation(ws.n)[: max(3, ws.n // 5)].astype(np.int64)
            pairs, _ = R.create_edges(ws, ws.sum_S, src, seeds[0])
            store["list_sources"] = src
            store["edges_list"] = pairs
        np.savez_compressed(os.path.join(OUT, f"edges_{name}.npz"), **store)
        meta[name] = {"n": int(w.size), "seeds": seeds}

    # ---- UCP plans and C_u bit patterns (plan_ucp_oracle, plan_ucp SPMD) ----
    plans = {}
    for t in range(12):
        n = int(rng.integers(50, 3000))
        w = np.sort(rng.uniform(0.1, 6.0, n))[::-1].copy()
        ws = R.weight_sequence(w)
        entry = {"w": w.tolist()}
        for P in (1, 2, 3, 4, 8, 16, 64):
            b = R.plan_ucp_oracle(ws, P)
            spmd = R.plan_ucp_spmd(ws, P)
            assert np.array_equal(b, spmd)
            entry[f"P{P}"] = b.tolist()
        plans[f"rand{t}"] = entry
    for t in range(3):  # dominant node -> empty partitions (acceptance.cpp:145-166)
        w = np.ones(60 + t)
        w[0] = 4000.0
        ws = R.weight_sequence(w)
        entry = {"w": w.tolist()}
        for P in (2, 3, 4, 8, 16, 64):
            entry[f"P{P}"] = R.plan_ucp_oracle(ws, P).tolist()
        plans[f"dominant{t}"] = entry
    with open(os.path.join(OUT, "plans.json"), "w") as fh:
        json.dump(plans, fh)

    # C_u bit patterns for a continuous power law at G in {1,2,4,8}
    ws = R.synth_powerlaw(100000, 2.5, 10.0, 1000.0, 1)
    store = {"w": ws.weights, "S": np.array([ws.sum_S])}
    for P in (1, 2, 4, 8):
        cum, bw, bc = R.global_cum_costs(ws, P)
        store[f"cum_P{P}"] = cum.view(np.uint64)
        store[f"bw_P{P}"] = bw.view(np.uint64)
        store[f"bc_P{P}"] = bc.view(np.uint64)
        store[f"plan_P{P}"] = R.plan_ucp_oracle(ws, P)
    np.savez_compressed(os.path.join(OUT, "costs_pl1e5.npz"), **store)

    # ---- scalars: skip_length, node_cost, blocked_sum, C1 headline ---------
    scal = {}
    pr = rng.uniform(1e-9, 1 - 1e-9, size=(2000, 2))
    scal["skip"] = [[p, r, R.skip_length(p, r)] for p, r in pr]
    ws = R.synth_powerlaw(1000000, 2.5, 10.0, 1000.0, 1)
    cnt, cks, _ = R.fold_edges_range(ws, ws.sum_S, 0, ws.n, 7)
    scal["c1_continuous"] = {
        "recipe": "synth_powerlaw(1e6, 2.5, 10, 1000, seed=1), generation seed 7",
        "S_bits": int(np.array([ws.sum_S]).view(np.uint64)[0]),
        "edges": cnt,
        "checksum": cks,
        "plan_P8": R.plan_ucp_oracle(ws, 8).tolist(),
        "plan_P2": R.plan_ucp_oracle(ws, 2).tolist(),
        "plan_P4": R.plan_ucp_oracle(ws, 4).tolist(),
    }
    ws = R.synth_constant(10000000, 50.0)
    scal["c2_S_bits"] = int(np.array([ws.sum_S]).view(np.uint64)[0])
    with open(os.path.join(OUT, "scalars.json"), "w") as fh:
        json.dump(scal, fh)
    with open(os.path.join(OUT, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
