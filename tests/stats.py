"""Exact FP64 expected-degree statistics for Chung–Lu graphs (test helpers).

E_i = sum_{v != i} min(w_i w_v / S, 1),  Var_i = sum_{v != i} p (1 - p),
computed in O(n log n) from the sorted weights: for node i the partners with
p >= 1 are the prefix w_v >= S / w_i (SURVEY.md §8(d) correctness gate 3).
"""
import numpy as np


def expected_degrees(w: np.ndarray, S: float, nodes: np.ndarray):
    w = np.asarray(w, np.float64)
    n = w.size
    nodes = np.asarray(nodes, np.int64)
    cw = np.concatenate([[0.0], np.cumsum(w)])
    cw2 = np.concatenate([[0.0], np.cumsum(w * w)])
    wi = w[nodes]
    E = np.zeros(nodes.size)
    V = np.zeros(nodes.size)
    if S <= 0:
        return E, V
    pos = wi > 0
    with np.errstate(divide="ignore"):
        thr = np.where(pos, S / np.where(pos, wi, 1.0), np.inf)
    # saturated partners form the prefix [0, m): w_v * w_i / S >= 1
    m = np.searchsorted(-w, -thr, side="right").astype(np.int64)
    for _ in range(3):  # exact FP64 boundary, as the generators evaluate it
        dec = (m > 0) & ~(w[np.maximum(m - 1, 0)] * wi / S >= 1.0)
        m = np.where(dec, m - 1, m)
        inc = (m < n) & (w[np.minimum(m, n - 1)] * wi / S >= 1.0)
        m = np.where(inc, m + 1, m)
    m = np.where(pos, m, 0)
    in_sat = nodes < m
    sat = m - in_sat
    mass = cw[n] - cw[m] - np.where(in_sat, 0.0, wi)
    mass2 = cw2[n] - cw2[m] - np.where(in_sat, 0.0, wi * wi)
    e_uns = wi * mass / S
    E = np.where(pos, sat + e_uns, 0.0)
    V = np.where(pos, e_uns - wi * wi * mass2 / (S * S), 0.0)
    return E, V


def chi2_z(obs: np.ndarray, E: np.ndarray, V: np.ndarray) -> tuple[float, int]:
    """(chi^2 - k) / sqrt(2k) over nodes with Var > 0."""
    ok = V > 1e-12
    k = int(ok.sum())
    chi2 = float(np.sum((obs[ok] - E[ok]) ** 2 / V[ok]))
    return (chi2 - k) / np.sqrt(2 * k), k


def total_edge_z(total: int, w: np.ndarray, S: float) -> float:
    """Total edge count vs sum_{u<v} min(p,1) with the exact Bernoulli variance."""
    nodes = np.arange(w.size)
    E, V = expected_degrees(w, S, nodes)
    mean = E.sum() / 2.0
    var = V.sum() / 2.0
    return (total - mean) / np.sqrt(var)


def mix64_np(z):
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def edge_hash_np(u, v):
    """The fold checksum's per-edge term (common.cuh edge_hash)."""
    with np.errstate(over="ignore"):
        z = ((u.astype(np.uint64) << np.uint64(32)) | v.astype(np.uint64)) * np.uint64(0x9E3779B97F4A7C15)
        z ^= z >> np.uint64(32)
        z *= np.uint64(0xD6E8FEB86659FD93)
        return z ^ (z >> np.uint64(32))


def checksum(pairs: np.ndarray) -> int:
    """Sum over edges of edge_hash(u, v) mod 2^64 (the streaming fold's checksum)."""
    return int(edge_hash_np(pairs[:, 0], pairs[:, 1]).sum(dtype=np.uint64))
