"""Generate the golden fixtures from the REFERENCE ITSELF.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It loads oracle/_ref/libhgr_ref.so (the unmodified reference headers compiled
behind a C ABI by oracle/Makefile) and records, for the inputs the reference's
own tests use (same seeds, libstdc++-exact mt19937 draws), the reference's
outputs. Small cases are stored in full (golden.npz); the BASELINE-sized CPU
config (513x513 fp64) and larger cases are stored as SHA-256 digests of the
output bytes plus sampled entries (golden_digests.json).

Nothing on the GPU box reads /root/reference; these files are the pinned record.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
import oracle  # noqa: E402
from oracle import random_coords as rc, random_values as rv  # noqa: E402
from tests.synthetic import smooth_field  # noqa: E402


def cases():
    """(name, shape, coords or None, dtype, input) mirroring the reference tests."""
    yield "quadratic_5", (5,), None, np.float64, np.array([6, 2, 0, 0, 2.0])
    # test_refactor.cpp:48-75 (dense-projection pipeline)
    yield "pipeline_1d", (9,), [rc(9, 2001)], np.float64, rv(9, 2002)
    yield "pipeline_2d", (5, 9), [rc(5, 2003), rc(9, 2004)], np.float64, rv(45, 2005).reshape(5, 9)
    yield ("pipeline_3d", (5, 5, 5), [rc(5, 2006), rc(5, 2007), rc(5, 2008)], np.float64,
           rv(125, 2009).reshape(5, 5, 5))
    # test_refactor.cpp:77-99 (affine)
    c0, c1 = rc(17, 2101), rc(9, 2102)
    yield "affine_17x9", (17, 9), [c0, c1], np.float64, 2.0 * c0[:, None] - 0.75 * c1[None, :] + 4.0
    # test_refactor.cpp:101-126 (round trips)
    yield "roundtrip_17cube", (17, 17, 17), None, np.float64, rv(17 ** 3, 2201).reshape(17, 17, 17)
    yield "roundtrip_33x17_nu", (33, 17), [rc(33, 2202), rc(17, 2203)], np.float64, rv(561, 2204).reshape(33, 17)
    yield "roundtrip_33sq_f32", (33, 33), None, np.float32, rv(1089, 2205).reshape(33, 33).astype(np.float32)
    # linearity / prefix / cascade / gather (test_refactor.cpp:128-273)
    yield "linear_u_9cube", (9, 9, 9), None, np.float64, rv(729, 2301).reshape(9, 9, 9)
    yield "linear_v_9cube", (9, 9, 9), None, np.float64, rv(729, 2302).reshape(9, 9, 9)
    yield "prefix_17sq", (17, 17), None, np.float64, rv(289, 2401).reshape(17, 17)
    yield "cascade_9x9_nu", (9, 9), [rc(9, 2501), rc(9, 2502)], np.float64, rv(81, 2503).reshape(9, 9)
    x = (np.arange(33) - 16.0) / 8.0
    yield "gauss_33sq", (33, 33), None, np.float64, np.exp(-(x[:, None] ** 2 + x[None, :] ** 2))
    yield "gather_9x5", (9, 5), None, np.float64, rv(45, 2601).reshape(9, 5)
    yield "passthrough_2", (2,), [np.array([0.0, 1.0])], np.float64, np.array([3.5, -1.25])
    yield "aniso_3x5x9_f32", (3, 5, 9), None, np.float32, rv(135, 77).reshape(3, 5, 9).astype(np.float32)


def digest_cases():
    yield "config0_513sq_f64", (513, 513), None, np.float64, smooth_field((513, 513), np.float64, 12345)
    yield "smooth_65cube_f32", (65, 65, 65), None, np.float32, smooth_field((65, 65, 65), np.float32, 12345)
    coords = [rc(33, 9001), rc(65, 9002), rc(129, 9003)]
    yield ("smooth_33x65x129_nu_f64", (33, 65, 129), coords, np.float64,
           smooth_field((33, 65, 129), np.float64, 12345))


def main():
    oracle.build()
    R = oracle.Oracle("reference")
    out = {}
    for name, shape, coords, dt, u in cases():
        u = np.asarray(u, dtype=dt).reshape(shape)
        pyr = R.decompose(u, coords)
        out[f"{name}/input"] = u
        out[f"{name}/decompose"] = pyr
        L = R.levels(shape, coords)
        for m in range(L + 1):
            out[f"{name}/recompose_{m}"] = R.recompose(pyr, m, coords)
        if coords is not None:
            for d, c in enumerate(coords):
                out[f"{name}/coords_{d}"] = c
        for cls in range(L + 1):
            out[f"{name}/class_{cls}"] = R.extract_class(pyr, cls, coords)
    # single-level known answers (test_correction.cpp:201-252, test_transforms.cpp:54-59)
    for n in (5, 9, 17):
        c = rc(n, 500 + n)
        v = rv(n, 600 + n)
        coeffs = np.where(np.arange(n) % 2 == 1, v, 0.0)
        L = R.levels((n,), [c])
        out[f"correction_1d_{n}/coords_0"] = c
        out[f"correction_1d_{n}/coeffs"] = coeffs
        out[f"correction_1d_{n}/z"] = R.compute_correction(coeffs, (n,), L, [c])
    for n in (5, 9):
        c0, c1 = rc(n, 700 + n), rc(n, 800 + n)
        v = rv(n * n, 900 + n).reshape(n, n)
        i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        coeffs = np.where((i % 2 == 1) | (j % 2 == 1), v, 0.0)
        L = R.levels((n, n), [c0, c1])
        out[f"correction_2d_{n}/coords_0"] = c0
        out[f"correction_2d_{n}/coords_1"] = c1
        out[f"correction_2d_{n}/coeffs"] = coeffs
        out[f"correction_2d_{n}/z"] = R.compute_correction(coeffs, (n, n), L, [c0, c1])
    for n in (5, 9, 33, 257, 1025):
        h = np.diff(rc(n, n + 7))
        v = rv(n, n + 11)
        out[f"masstrans_{n}/h"] = h
        out[f"masstrans_{n}/v"] = v
        out[f"masstrans_{n}/out"] = R.masstrans_apply(v, h)
        out[f"mass_{n}/out"] = R.mass_apply(v, h)
    for n in (2, 5, 65, 257, 1025):
        h = np.diff(rc(n, n))
        v = rv(n, n + 1)
        rhs = R.mass_apply(v, h)
        out[f"thomas_{n}/h"] = h
        out[f"thomas_{n}/v"] = v
        out[f"thomas_{n}/rhs"] = rhs
        out[f"thomas_{n}/out"] = R.thomas_solve(rhs, h)
    np.savez_compressed(HERE / "golden.npz", **out)

    digests = {}
    for name, shape, coords, dt, u in digest_cases():
        pyr = R.decompose(u, coords)
        L = R.levels(shape, coords)
        back = R.recompose(pyr, L, coords)
        half = R.recompose(pyr, L // 2, coords)
        rng = np.random.default_rng(0)
        idx = rng.integers(0, u.size, 64)
        digests[name] = {
            "shape": list(shape), "dtype": np.dtype(dt).name, "seed": 12345,
            "coords_seeds": [9001, 9002, 9003] if coords else None,
            "input_sha256": hashlib.sha256(u.tobytes()).hexdigest(),
            "decompose_sha256": hashlib.sha256(pyr.tobytes()).hexdigest(),
            "recompose_full_sha256": hashlib.sha256(back.tobytes()).hexdigest(),
            "recompose_half_sha256": hashlib.sha256(half.tobytes()).hexdigest(),
            "sample_index": idx.tolist(),
            "decompose_sample": pyr.reshape(-1)[idx].astype(np.float64).tolist(),
            "recompose_full_sample": back.reshape(-1)[idx].astype(np.float64).tolist(),
            "max_abs_input": float(np.abs(u).max()),
        }
    (HERE / "golden_digests.json").write_text(json.dumps(digests, indent=1))
    print(f"wrote {len(out)} arrays, {len(digests)} digests")


if __name__ == "__main__":
    main()
