"""Seeded synthetic input generators shared by the tests, the oracle and bench.py.

This module holds NONE of the method's arithmetic (no schedule, no rotation, no
gradient). It only turns (seed, tensor_id, element index) into numbers with a
counter-based hash (SplitMix64 finaliser), so any rank, any column shard and the
CPU oracle can regenerate exactly the same values independently.

Recipe:
  * theta ~ U(-pi, pi) in fp32           ("unrestricted");
    parity tests also use U(-8 pi, 8 pi) and special values (+-2 pi, 1e3, -1e4, ...)
  * X, dY, Gamma ~ N(0, 1) in fp32        (Box-Muller on two hashed uniforms)
  * element (row, col) of an n x m tensor is hashed from its flat row-major index
    row * m_total + col, so a column shard [c0, c1) is reproducible on its own.
"""
from __future__ import annotations

import numpy as np

_MASK = np.uint64(0xFFFFFFFFFFFFFFFF)

# tensor ids (stable, part of the recipe)
TID_THETA = 1
TID_X = 2
TID_DY = 3
TID_GAMMA = 4
TID_MASK = 5


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _MASK
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _MASK
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _MASK
        return z ^ (z >> np.uint64(31))


def _keys(seed: int, tid: int, idx: np.ndarray, stream: int = 0) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = _splitmix64(np.asarray([(seed * 0x100000001B3 + tid * 0x9E37 + stream * 0x7F4A7C15) & 0xFFFFFFFFFFFFFFFF],
                                      dtype=np.uint64))[0]
        return _splitmix64((idx.astype(np.uint64) * np.uint64(0xD1B54A32D192ED03) + base) & _MASK)


def uniform01(seed: int, tid: int, idx: np.ndarray, stream: int = 0) -> np.ndarray:
    """fp64 uniforms in [0, 1) with 53 random bits, one per index."""
    k = _keys(seed, tid, idx, stream)
    return (k >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def theta(n_angles: int, seed: int = 0, half_range: float = np.pi) -> np.ndarray:
    """fp32 angles ~ U(-half_range, half_range), length n_angles, block-major flat order.

    The default half_range = pi is the bench recipe; the paper's angles are unrestricted reals
    (PAPER.md:184), so the parity tests also draw wide ranges (e.g. half_range = 8 pi)."""
    u = uniform01(seed, TID_THETA, np.arange(n_angles, dtype=np.uint64))
    return ((2.0 * u - 1.0) * half_range).astype(np.float32)


def normal_matrix(n: int, m_total: int, seed: int, tid: int, col0: int = 0, col1: int | None = None,
                  dtype=np.float32) -> np.ndarray:
    """N(0,1) n x (col1-col0) block of the n x m_total tensor `tid` (row-major)."""
    if col1 is None:
        col1 = m_total
    rows = np.arange(n, dtype=np.uint64)[:, None]
    cols = np.arange(col0, col1, dtype=np.uint64)[None, :]
    idx = rows * np.uint64(m_total) + cols
    u1 = uniform01(seed, tid, idx, 0)
    u2 = uniform01(seed, tid, idx, 1)
    r = np.sqrt(-2.0 * np.log1p(-u1))          # 1-u1 in (0, 1]
    return (r * np.cos(2.0 * np.pi * u2)).astype(dtype)


def random_mask(n_angles: int, keep_prob: float, seed: int = 0) -> np.ndarray:
    """uint8 mask (1 = free angle, 0 = pinned to zero), i.i.d. Bernoulli(keep_prob)."""
    u = uniform01(seed, TID_MASK, np.arange(n_angles, dtype=np.uint64))
    return (u < keep_prob).astype(np.uint8)
