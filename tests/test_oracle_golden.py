"""CPU suite: pin the oracles before trusting them.

* the C restatement (oracle/hgr_oracle.c) reproduces every golden vector the
  reference produced (tests/golden/, made by make_golden.py from the reference
  itself) -- bit for bit, both being compiled without FMA contraction;
* the reference's own hard-coded known answers (test_*.cpp) hold;
* the independent dense Galerkin oracle (oracle/galerkin.py, restating
  oracle_helpers.hpp) agrees with the golden corrections/pipelines to 1e-10,
  as test_correction.cpp:201-252 and test_refactor.cpp:48-75 require.
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from oracle import galerkin
from tests.synthetic import smooth_field

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(GOLD / "golden.npz"))


def _cases(golden):
    names = sorted({k.split("/")[0] for k in golden if k.endswith("/decompose")})
    for name in names:
        u = golden[f"{name}/input"]
        coords = None
        if f"{name}/coords_0" in golden:
            coords = [golden[f"{name}/coords_{d}"] for d in range(u.ndim)]
        yield name, u, coords


def test_golden_present(golden):
    assert len(list(_cases(golden))) >= 15


@pytest.mark.parametrize("kind", ["port", "reference"])
def test_oracle_matches_golden_bitwise(golden, kind):
    if kind == "reference" and not oracle.available("reference"):
        pytest.skip("reference oracle not built")
    O = oracle.Oracle(kind)
    for name, u, coords in _cases(golden):
        pyr = O.decompose(u, coords)
        assert np.array_equal(pyr, golden[f"{name}/decompose"]), name
        L = O.levels(u.shape, coords)
        for m in range(L + 1):
            assert np.array_equal(O.recompose(pyr, m, coords), golden[f"{name}/recompose_{m}"]), (name, m)
        for cls in range(L + 1):
            assert np.array_equal(O.extract_class(pyr, cls, coords), golden[f"{name}/class_{cls}"])


def test_port_single_level_golden(golden, port):
    for n in (5, 9, 17):
        c = golden[f"correction_1d_{n}/coords_0"]
        z = port.compute_correction(golden[f"correction_1d_{n}/coeffs"], (n,), port.levels((n,), [c]), [c])
        assert np.array_equal(z, golden[f"correction_1d_{n}/z"])
    for n in (5, 9):
        cs = [golden[f"correction_2d_{n}/coords_{d}"] for d in range(2)]
        z = port.compute_correction(golden[f"correction_2d_{n}/coeffs"], (n, n), port.levels((n, n), cs), cs)
        assert np.array_equal(z, golden[f"correction_2d_{n}/z"])
    for n in (5, 9, 33, 257, 1025):
        h, v = golden[f"masstrans_{n}/h"], golden[f"masstrans_{n}/v"]
        assert np.array_equal(port.masstrans_apply(v, h), golden[f"masstrans_{n}/out"])
        assert np.array_equal(port.mass_apply(v, h), golden[f"mass_{n}/out"])
    for n in (2, 5, 65, 257, 1025):
        h, rhs = golden[f"thomas_{n}/h"], golden[f"thomas_{n}/rhs"]
        z = port.thomas_solve(rhs, h)
        assert np.array_equal(z, golden[f"thomas_{n}/out"])
        # test_correction.cpp:120-146: recovers v to 1e-12
        assert np.abs(z - golden[f"thomas_{n}/v"]).max() <= 1e-12


def test_port_digests(port):
    """BASELINE config 0 (513x513 fp64) and two larger cases, pinned by digest."""
    dig = json.loads((GOLD / "golden_digests.json").read_text())
    for name, d in dig.items():
        shape = tuple(d["shape"])
        dt = np.dtype(d["dtype"]).type
        coords = None
        if d["coords_seeds"]:
            coords = [oracle.random_coords(n, s) for n, s in zip(shape, d["coords_seeds"])]
        u = smooth_field(shape, dt, d["seed"])
        assert hashlib.sha256(u.tobytes()).hexdigest() == d["input_sha256"], name
        pyr = port.decompose(u, coords)
        assert hashlib.sha256(pyr.tobytes()).hexdigest() == d["decompose_sha256"], name
        L = port.levels(shape, coords)
        back = port.recompose(pyr, L, coords)
        assert hashlib.sha256(back.tobytes()).hexdigest() == d["recompose_full_sha256"], name
        half = port.recompose(pyr, L // 2, coords)
        assert hashlib.sha256(half.tobytes()).hexdigest() == d["recompose_half_sha256"], name


def test_reference_known_answers(port):
    """Hard-coded expectations from the reference's own tests."""
    # test_refactor.cpp:31-46
    np.testing.assert_allclose(port.decompose(np.array([6, 2, 0, 0, 2.0])), [3.5, -1, -4, -1, -0.5],
                               rtol=1e-14)
    # test_transforms.cpp:30-35, 47-52, 54-59, 78-83
    assert list(port.interpolate_to_fine(np.array([6.0, 0, 2]), (5,), 2)) == [6, 3, 0, 1, 2]
    assert abs(port.interpolate_to_fine(np.array([0.0, 3]), (3,), 1, [np.array([0, 1, 3.0])])[1] - 1) < 1e-15
    assert list(port.compute_coefficients(np.array([6.0, 2, 0, 0, 2]), (5,), 2)) == [0, -1, 0, -1, 0]
    bump = np.zeros((3, 3)); bump[1, 1] = 1
    assert np.array_equal(port.compute_coefficients(bump, (3, 3), 1), bump)
    # test_correction.cpp:35-68
    h = np.ones(4)
    assert list(port.mass_apply(np.ones(5), h)) == [3, 6, 6, 6, 3]
    assert list(port.mass_apply(np.array([0, -1, 0, -1, 0.0]), h)) == [-1, -4, -2, -4, -1]
    assert list(port.transfer_apply(np.array([0, -1, 0, -1, 0.0]), h)) == [-0.5, -1, -0.5]
    assert list(port.transfer_apply(np.array([0, 3, 0.0]), np.array([1.0, 2]))) == [2, 1]
    assert list(port.masstrans_apply(np.array([0, -1, 0, -1, 0.0]), h)) == [-3, -6, -3]
    np.testing.assert_allclose(port.thomas_solve(np.array([-3.0, -6, -3]), np.array([2.0, 2])), [-0.5] * 3,
                               rtol=1e-14)
    # test_correction.cpp:153-175
    np.testing.assert_allclose(port.compute_correction(np.array([0, -1, 0, -1, 0.0]), (5,), 2), [-0.5] * 3,
                               rtol=1e-14)
    c1 = np.array([0, -1, 0, -1, 0.0])
    np.testing.assert_allclose(port.compute_correction(np.outer(c1, c1), (5, 5), 2), np.full((3, 3), 0.25),
                               rtol=1e-13)
    with pytest.raises(oracle.OracleError, match="zero at coarse"):
        port.compute_correction(np.array([1, -1, 0, -1, 0.0]), (5,), 2)
    # test_grid_hierarchy / class counts (test_refactor.cpp:207-215)
    assert port.levels((513,)) == 9 and port.levels((513, 513, 513)) == 9 and port.levels((33, 33, 33)) == 5
    assert sum(port.class_node_count((513,), c) for c in range(10)) == 513
    with pytest.raises(oracle.OracleError, match="2\\^k\\+1"):
        port.levels((6,))
    with pytest.raises(oracle.OracleError, match="non-finite"):
        port.decompose(np.array([0, 1, np.nan, 3, 4.0]))
    with pytest.raises(oracle.OracleError, match="class index out of range"):
        port.recompose(np.zeros(5), 3)


def test_dense_galerkin_agrees(golden):
    """oracle/galerkin.py (independent) vs the golden reference outputs, 1e-10."""
    for n in (5, 9, 17):
        c = golden[f"correction_1d_{n}/coords_0"]
        z = galerkin.galerkin_correction([c], galerkin.coarsen([c]), golden[f"correction_1d_{n}/coeffs"])
        assert np.abs(z - golden[f"correction_1d_{n}/z"].reshape(-1)).max() <= 1e-10
    for n in (5, 9):
        cs = [golden[f"correction_2d_{n}/coords_{d}"] for d in range(2)]
        z = galerkin.galerkin_correction(cs, galerkin.coarsen(cs), golden[f"correction_2d_{n}/coeffs"])
        assert np.abs(z - golden[f"correction_2d_{n}/z"].reshape(-1)).max() <= 1e-10
    for name in ("pipeline_1d", "pipeline_2d", "pipeline_3d"):
        u = golden[f"{name}/input"]
        cs = [golden[f"{name}/coords_{d}"] for d in range(u.ndim)]
        want = galerkin.decompose(cs, u)
        assert np.abs(want - golden[f"{name}/decompose"]).max() <= 1e-10


def test_golden_properties(golden):
    """Property checks on the reference outputs themselves (test_refactor.cpp)."""
    # affine -> class 0 only (test_refactor.cpp:77-99)
    u = golden["affine_17x9/input"]
    peak = np.abs(u).max()
    for cls in range(1, 4):
        assert np.abs(golden[f"affine_17x9/class_{cls}"]).max() <= 1e-12 * peak
    # linearity (test_refactor.cpp:128-157)
    a, b = 1.75, -2.5
    ru, rv = golden["linear_u_9cube/decompose"], golden["linear_v_9cube/decompose"]
    port = oracle.Oracle("port")
    rm = port.decompose(a * golden["linear_u_9cube/input"] + b * golden["linear_v_9cube/input"])
    assert np.abs(rm - (a * ru + b * rv)).max() <= 1e-11 * 4.25
    # monotone error decline (test_refactor.cpp:189-205)
    g = golden["gauss_33sq/input"]
    prev = np.inf
    for m in range(6):
        e = np.sqrt(((golden[f"gauss_33sq/recompose_{m}"] - g) ** 2).sum() / (g ** 2).sum())
        assert e <= prev + 1e-15
        prev = e
    assert prev <= 1e-12


def test_rng_matches_libstdcxx(ref):
    import ctypes as C
    for seed in (1, 2002, 9001):
        out = np.zeros(50)
        ref.lib.hgrref_random_values(C.c_size_t(50), C.c_uint(seed), out.ctypes.data_as(C.c_void_p))
        assert np.array_equal(out, oracle.random_values(50, seed))
        ref.lib.hgrref_random_coords(C.c_size_t(50), C.c_uint(seed), out.ctypes.data_as(C.c_void_p))
        assert np.array_equal(out, oracle.random_coords(50, seed))
