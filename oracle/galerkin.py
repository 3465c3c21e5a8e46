"""TEST INFRASTRUCTURE ONLY -- independent dense oracle, numpy restatement of
the reference's Eigen-based test helpers (proj/tests/oracle_helpers.hpp).

* hat / hat_product_integral / mass_matrix / mixed_mass  (oracle_helpers.hpp:19-68):
  Gram matrices of the piecewise-linear hat basis by Simpson quadrature on the
  fine grid (exact for products of piecewise-linear functions).
* galerkin_correction (:81-91): L2 projection of the fine piecewise-multilinear
  coefficient function onto the coarse space via dense Kronecker systems.
* interpolate (:110-156), coarsen (:103-108), decompose (:160-226): a
  compact-array multilevel decomposition built from the above.

It shares no code path with the library or with oracle/hgr_oracle.c: weights
come straight from coordinates and the correction from dense linear algebra.
"""
from __future__ import annotations

import numpy as np


def hat(grid, i, t):
    grid = np.asarray(grid)
    out = np.zeros_like(np.asarray(t, dtype=np.float64))
    if i > 0:
        m = (t >= grid[i - 1]) & (t <= grid[i])
        out = np.where(m, (t - grid[i - 1]) / (grid[i] - grid[i - 1]), out)
    if i + 1 < len(grid):
        m = (t >= grid[i]) & (t <= grid[i + 1]) & (out == 0)
        out = np.where(m, (grid[i + 1] - t) / (grid[i + 1] - grid[i]), out)
    return out


def hat_product_integral(quad, ga, a, gb, b):
    quad = np.asarray(quad)
    x0, x1 = quad[:-1], quad[1:]
    xm = 0.5 * (x0 + x1)
    f0 = hat(ga, a, x0) * hat(gb, b, x0)
    fm = hat(ga, a, xm) * hat(gb, b, xm)
    f1 = hat(ga, a, x1) * hat(gb, b, x1)
    return float(np.sum((x1 - x0) / 6.0 * (f0 + 4.0 * fm + f1)))


def mass_matrix(grid):
    n = len(grid)
    return np.array([[hat_product_integral(grid, grid, i, grid, j) for j in range(n)] for i in range(n)])


def mixed_mass(coarse, fine):
    return np.array([[hat_product_integral(fine, coarse, i, fine, j) for j in range(len(fine))]
                     for i in range(len(coarse))])


def galerkin_correction(fine, coarse, coeffs):
    gram = np.eye(1)
    mixed = np.eye(1)
    for f, c in zip(fine, coarse):
        gram = np.kron(gram, mass_matrix(c))
        mixed = np.kron(mixed, mixed_mass(c, f))
    return np.linalg.solve(gram, mixed @ np.asarray(coeffs, dtype=np.float64).reshape(-1))


def coarsen(coords):
    return [np.asarray(c)[::2] for c in coords]


def interpolate(fine_coords, coarse_values):
    rank = len(fine_coords)
    fe = [len(c) for c in fine_coords]
    ce = [(n - 1) // 2 + 1 for n in fe]
    f = fe + [1] * (3 - rank)
    c = ce + [1] * (3 - rank)
    fc = list(fine_coords) + [np.zeros(1)] * (3 - rank)
    cv = np.asarray(coarse_values, dtype=np.float64).reshape(c)
    out = np.zeros(f)
    for i0 in range(f[0]):
        for i1 in range(f[1]):
            for i2 in range(f[2]):
                idx = (i0, i1, i2)
                acc = 0.0
                for corner in range(8):
                    w, at, skip = 1.0, [0, 0, 0], False
                    for d in range(3):
                        q = idx[d] // 2
                        if idx[d] % 2 == 0:
                            if corner & (1 << d):
                                skip = True
                            at[d] = q
                            continue
                        x, xa, xb = fc[d][idx[d]], fc[d][idx[d] - 1], fc[d][idx[d] + 1]
                        if corner & (1 << d):
                            at[d] = q + 1
                            w *= (x - xa) / (xb - xa)
                        else:
                            at[d] = q
                            w *= (xb - x) / (xb - xa)
                    if not skip:
                        acc += w * cv[tuple(at)]
                out[idx] = acc
    return out.reshape(fe)


def decompose(coords, data):
    """Compact-array multilevel decomposition (oracle_helpers.hpp:160-226)."""
    rank = len(coords)
    min_side = min(len(c) for c in coords)
    levels, s = 0, min_side - 1
    while s > 1:
        levels += 1
        s //= 2
    level_coords = [list(coords)]
    for _ in range(levels):
        level_coords.append(coarsen(level_coords[-1]))
    classes = [None] * (levels + 1)
    cur = np.asarray(data, dtype=np.float64).reshape([len(c) for c in coords])
    for l in range(levels, 0, -1):
        fc = level_coords[levels - l]
        sl = tuple(slice(None, None, 2) for _ in range(rank))
        coarse_vals = cur[sl].copy()
        interp = interpolate(fc, coarse_vals)
        refined = np.zeros(cur.shape, dtype=bool)
        for d in range(rank):
            shp = [1] * rank
            shp[d] = cur.shape[d]
            refined |= (np.arange(cur.shape[d]) % 2 == 1).reshape(shp)
        coeffs = np.where(refined, cur - interp, 0.0)
        classes[l] = (cur - interp)[refined]
        z = galerkin_correction(fc, level_coords[levels - l + 1], coeffs)
        cur = coarse_vals + z.reshape(coarse_vals.shape)
    classes[0] = cur.reshape(-1)
    shape = [len(c) for c in coords]
    out = np.zeros(shape)
    for cls in range(levels + 1):
        stride = 1 << (levels - cls)
        sl = tuple(slice(None, None, stride) for _ in range(rank))
        view = out[sl]
        if cls == 0:
            view[...] = classes[0].reshape(view.shape)
        else:
            mask = np.zeros(view.shape, dtype=bool)
            for d in range(rank):
                shp = [1] * rank
                shp[d] = view.shape[d]
                mask |= (np.arange(view.shape[d]) % 2 == 1).reshape(shp)
            view[mask] = classes[cls]
        out[sl] = view
    return out
