"""Seeded input vectors by GLOBAL panel id (no arithmetic of the method): a counter-based
generator, so every rank of a distributed run draws exactly its own entries of the same vector
without materialising the whole of it (SplitMix64 -> two uniforms -> Box-Muller)."""
from __future__ import annotations

import numpy as np

_M1, _M2, _M3 = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)


def _splitmix64(z):
    z = (z + _M1).astype(np.uint64)
    z = ((z ^ (z >> np.uint64(30))) * _M2).astype(np.uint64)
    z = ((z ^ (z >> np.uint64(27))) * _M3).astype(np.uint64)
    return z ^ (z >> np.uint64(31))


def normal_by_id(ids, seed: int = 0):
    """N(0, 1) samples, one per id (int64 array), identical for the same (id, seed) on every rank."""
    ids = np.asarray(ids, np.uint64)
    with np.errstate(over="ignore"):
        base = (ids * np.uint64(2) + np.uint64(seed) * np.uint64(0x632BE59BD9B4E019)).astype(np.uint64)
        u1 = (_splitmix64(base) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        u2 = (_splitmix64(base + np.uint64(1)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
