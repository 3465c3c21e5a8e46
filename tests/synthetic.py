"""Deterministic synthetic inputs, host side.

u[i,j,k] = sin(0.21 i) cos(0.13 j) + 0.5 sin(0.07 k) + 1e-3 * eta(flat)
(the reference's "smooth" pattern, proj/tests/gen_raw.cpp:46-47, plus a small
counter-based noise eta in [-1, 1) from splitmix64(seed + flat)). Rank < 3
drops the missing index terms (1D: 0.5 sin(0.07 k); 2D: sin(0.21 i) cos(0.13 j)
... see _factors). Computed in float64, cast once to the target dtype. The
device generator (bench.py) builds the same 1D factor tables on the host and
combines them with IEEE-exact mul/add, so both sides are bitwise identical.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def noise(n: int, seed: int, start: int = 0) -> np.ndarray:
    flat = np.arange(start, start + n, dtype=np.uint64) + np.uint64(seed)
    r = (splitmix64(flat) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return r * 2.0 - 1.0


def factors(shape):
    """1D factor tables a(i), b(j), c(k) with u = a*b + c. The shape is padded
    on the right (as the reference pads, ndarray.hpp:90-94), so a missing j
    gives cos(0) = 1 and a missing k gives 0.5 sin(0) = 0: the missing index
    terms drop out (2D: sin(0.21 i) cos(0.13 j); 1D: sin(0.21 i))."""
    e = list(shape) + [1] * (3 - len(shape))
    i, j, k = (np.arange(n, dtype=np.float64) for n in e)
    return np.sin(0.21 * i), np.cos(0.13 * j), 0.5 * np.sin(0.07 * k)


def smooth_field(shape, dtype=np.float64, seed: int = 12345) -> np.ndarray:
    a, b, c = factors(shape)
    base = (a[:, None, None] * b[None, :, None]) + c[None, None, :]
    n = base.size
    u = base.reshape(-1) + 1e-3 * noise(n, seed)
    return u.reshape(shape).astype(dtype)
