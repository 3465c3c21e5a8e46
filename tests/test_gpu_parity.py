"""GPU parity tests: the CUDA path (through the C ABI) vs the CPU oracle on the
same seeded inputs. Tolerances are north_star's: max-abs <= 1e-12*max|u| for
fp64 and <= 1e-5*max|u| for fp32, for coefficients, recomposed data and the
round trip."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

TOL = {np.float64: 1e-12, np.float32: 1e-5}


def _hgr():
    import paper_2007_04457_b200 as hgr
    return hgr


def rel(a, b, scale):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max()) / scale


def make_grid(hgr, shape, nonuniform, seed=100):
    if not nonuniform:
        return hgr.GridHierarchy.uniform(list(shape)), None
    coords = [oracle.random_coords(n, seed + d) for d, n in enumerate(shape)]
    return hgr.GridHierarchy(coords), coords


SHAPES = [
    (5,), (9,), (1025,), (2,), (3,),
    (3, 3), (5, 5), (9, 5), (17, 33), (65, 65), (3, 9), (129, 17),
    (3, 3, 3), (5, 5, 5), (9, 5, 17), (17, 17, 17), (33, 33, 33), (65, 9, 5), (5, 9, 65),
    (33, 65, 17), (3, 5, 9), (2, 3, 5), (65, 65, 65),
]


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("nonuniform", [False, True], ids=["uniform", "nonuniform"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_decompose_recompose_vs_oracle(cuda, port, shape, nonuniform, dt):
    import torch
    hgr = _hgr()
    g, coords = make_grid(hgr, shape, nonuniform)
    rng = np.random.default_rng(hash((shape, nonuniform)) % 2**32)
    u = rng.uniform(-1, 1, shape).astype(dt)
    scale = float(np.abs(u).max())
    tol = TOL[dt]
    expect = port.decompose(u, coords)
    r = hgr.decompose(torch.from_numpy(u).to(cuda), g)
    got = r.data.cpu().numpy()
    assert rel(got, expect, scale) <= tol
    L = g.levels()
    for m in sorted({0, L // 2, L}):
        want = port.recompose(expect, m, coords)
        back = hgr.recompose(r, m).cpu().numpy()
        assert rel(back, want, scale) <= tol, f"recompose upto {m}"
    back = hgr.recompose(r, L).cpu().numpy()
    assert rel(back, u, scale) <= tol


def test_worked_quadratic(cuda):
    """test_refactor.cpp:31-46: [6,2,0,0,2] -> [3.5,-1,-4,-1,-0.5]."""
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy.uniform([5])
    r = hgr.decompose(torch.tensor([6, 2, 0, 0, 2], dtype=torch.float64, device=cuda), g)
    np.testing.assert_allclose(r.data.cpu().numpy(), [3.5, -1, -4, -1, -0.5], rtol=1e-14, atol=1e-14)
    cls2 = hgr.extract_class(r, 2).cpu().numpy()
    assert list(cls2) == [-1, -1]
    back = hgr.recompose(r, 2).cpu().numpy()
    np.testing.assert_allclose(back, [6, 2, 0, 0, 2], atol=1e-12 * 6)


def test_two_node_passthrough(cuda):
    """test_refactor.cpp:217-223."""
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy([[0.0, 1.0]])
    r = hgr.decompose(torch.tensor([3.5, -1.25], dtype=torch.float64, device=cuda), g)
    assert r.data.cpu().tolist() == [3.5, -1.25]
    assert hgr.recompose(r, 0).cpu().tolist() == [3.5, -1.25]
    assert hgr.extract_class(r, 0).cpu().tolist() == [3.5, -1.25]


def test_validation(cuda):
    """test_refactor.cpp:250-259 and test_grid_hierarchy.cpp:27-35."""
    import torch
    hgr = _hgr()
    with pytest.raises(hgr.HgrError, match="2\\^k\\+1"):
        hgr.GridHierarchy.uniform([6])
    g = hgr.GridHierarchy.uniform([5])
    with pytest.raises(hgr.HgrError):
        hgr.decompose(torch.zeros(4, dtype=torch.float64, device=cuda), g)
    bad = torch.tensor([0, 1, float("nan"), 3, 4], dtype=torch.float64, device=cuda)
    with pytest.raises(hgr.HgrError, match="non-finite"):
        hgr.decompose(bad, g)
    r = hgr.decompose(torch.tensor([1, 2, 3, 4, 5.0], dtype=torch.float64, device=cuda), g)
    with pytest.raises(hgr.HgrError, match="class index out of range"):
        hgr.recompose(r, 3)
    with pytest.raises(hgr.HgrError):
        hgr.recompose(r, -1)


def test_prefix_bit_identity(cuda):
    """test_refactor.cpp:159-172: recompose(r, m) == recompose(zeroed above m, m), bitwise."""
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy.uniform([17, 17])
    u = oracle.random_values(17 * 17, 2401).reshape(17, 17)
    r = hgr.decompose(torch.from_numpy(u).to(cuda), g)
    for m in range(g.levels() + 1):
        direct = hgr.recompose(r, m)
        zeroed = hgr.RefactoredArray(r.data.clone(), g)
        for cls in range(m + 1, g.levels() + 1):
            hgr.scatter_class(zeroed, cls, torch.zeros(g.class_node_count(cls), dtype=torch.float64, device=cuda))
        via = hgr.recompose(zeroed, m)
        assert torch.equal(direct, via)


def test_determinism(cuda):
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy.uniform([65, 33, 17])
    u = torch.rand(65, 33, 17, dtype=torch.float64, device=cuda)
    a = hgr.decompose(u, g).data
    b = hgr.decompose(u, g).data
    assert torch.equal(a, b)
    assert torch.equal(hgr.recompose(hgr.RefactoredArray(a, g), 3), hgr.recompose(hgr.RefactoredArray(b, g), 3))


@pytest.mark.parametrize("shape", [(9, 5), (17, 9, 5), (33,)], ids=str)
def test_extract_scatter_vs_oracle(cuda, port, shape):
    """refactor.hpp:134-170 packing order; test_refactor.cpp:261-273 duality."""
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy.uniform(list(shape))
    u = np.random.default_rng(3).uniform(-1, 1, shape)
    r = hgr.RefactoredArray(torch.from_numpy(u).to(cuda), g)
    copy = hgr.RefactoredArray(torch.zeros_like(r.data), g)
    for cls in range(g.levels() + 1):
        vals = hgr.extract_class(r, cls)
        assert np.array_equal(vals.cpu().numpy(), port.extract_class(u, cls))
        hgr.scatter_class(copy, cls, vals)
    assert torch.equal(copy.data, r.data)
    with pytest.raises(hgr.HgrError):
        hgr.scatter_class(copy, 0, torch.zeros(3, dtype=torch.float64, device=cuda))


def test_single_level_kats(cuda):
    """test_transforms.cpp:30-83 and test_correction.cpp:153-175 known answers."""
    hgr = _hgr()
    g = hgr.GridHierarchy([[0, 1, 2, 3, 4]])
    assert list(hgr.interpolate_to_fine(np.array([6.0, 0, 2]), g, 2)) == [6, 3, 0, 1, 2]
    assert list(hgr.compute_coefficients(np.array([6.0, 2, 0, 0, 2]), g, 2)) == [0, -1, 0, -1, 0]
    fine = hgr.apply_coefficients(np.array([6.0, 0, 2]), np.array([0.0, -1, 0, -1, 0]), g, 2)
    assert list(fine) == [6, 2, 0, 0, 2]
    gn = hgr.GridHierarchy([[0, 1, 3]])
    assert abs(hgr.interpolate_to_fine(np.array([0.0, 3]), gn, 1)[1] - 1.0) <= 1e-15
    g33 = hgr.GridHierarchy.uniform([3, 3])
    bump = np.zeros((3, 3)); bump[1, 1] = 1
    assert np.array_equal(hgr.compute_coefficients(bump, g33, 1), bump)
    z = hgr.compute_correction(np.array([0.0, -1, 0, -1, 0]), g, 2)
    np.testing.assert_allclose(z, [-0.5] * 3, rtol=1e-14)
    assert list(hgr.compute_correction(np.zeros(5), g, 2)) == [0, 0, 0]
    g55 = hgr.GridHierarchy.uniform([5, 5])
    c1 = np.array([0, -1, 0, -1, 0.0])
    coeffs = np.outer(c1, c1)
    np.testing.assert_allclose(hgr.compute_correction(coeffs, g55, 2), np.full((3, 3), 0.25), rtol=1e-13)
    with pytest.raises(hgr.HgrError, match="zero at coarse"):
        hgr.compute_correction(np.array([1.0, -1, 0, -1, 0]), g, 2)


def test_fiber_kats(cuda):
    """test_correction.cpp:35-68, 109-118."""
    hgr = _hgr()
    h = np.ones(4)
    assert list(hgr.mass_apply(np.ones(5), h)) == [3, 6, 6, 6, 3]
    assert list(hgr.mass_apply(np.array([0, -1, 0, -1, 0.0]), h)) == [-1, -4, -2, -4, -1]
    assert list(hgr.masstrans_apply(np.array([0, -1, 0, -1, 0.0]), h)) == [-3, -6, -3]
    z = hgr.thomas_solve(np.array([-3.0, -6, -3]), np.array([2.0, 2]))
    np.testing.assert_allclose(z, [-0.5] * 3, rtol=1e-14)


@pytest.mark.parametrize("n", [5, 9, 33, 257, 1025])
def test_fiber_ops_vs_oracle(cuda, port, n):
    hgr = _hgr()
    coords = oracle.random_coords(n, n + 7)
    h = np.diff(coords)
    v = oracle.random_values(n, n + 11)
    np.testing.assert_allclose(hgr.masstrans_apply(v, h), port.masstrans_apply(v, h), rtol=0, atol=1e-13)
    np.testing.assert_allclose(hgr.thomas_solve(v, h), port.thomas_solve(v, h), rtol=0, atol=1e-13)
    np.testing.assert_allclose(hgr.mass_apply(v, h), port.mass_apply(v, h), rtol=0, atol=1e-13)


FUSED_SHAPES = [(65, 65, 65), (33, 129, 65), (129, 33, 17), (17, 257, 129), (257, 257), (1025, 65),
                (65537,), (5, 65, 257), (9, 129, 33)]


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("nonuniform", [False, True], ids=["uniform", "nonuniform"])
@pytest.mark.parametrize("shape", FUSED_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_fused_levels_vs_oracle(cuda, port, shape, nonuniform, dt):
    """Sizes that take the fused level kernels (>= 4096 nodes per level)."""
    import torch
    hgr = _hgr()
    g, coords = make_grid(hgr, shape, nonuniform, seed=300)
    from tests.synthetic import smooth_field
    u = smooth_field(shape, dt, 12345)
    scale = float(np.abs(u).max())
    tol = TOL[dt]
    expect = port.decompose(u, coords)
    x = torch.from_numpy(u).to(cuda)
    plan = hgr.Plan(g, "f64" if dt == np.float64 else "f32")
    out = torch.empty_like(x)
    plan.decompose_into(x, out)
    plan.sync_status()
    assert torch.equal(x, torch.from_numpy(u).to(cuda)), "decompose_into must not modify its input"
    assert rel(out.cpu().numpy(), expect, scale) <= tol
    inplace = x.clone()
    plan.decompose_(inplace)
    plan.sync_status()
    assert rel(inplace.cpu().numpy(), expect, scale) <= tol
    L = g.levels()
    for m in sorted({0, L - 1, L}):
        back = torch.empty_like(x)
        plan.recompose_into(out, back, m)
        assert rel(back.cpu().numpy(), port.recompose(expect, m, coords), scale) <= tol, m
    same = out.clone()
    plan.recompose_into(same, same, L)  # in-place recompose
    assert rel(same.cpu().numpy(), u, scale) <= tol


def test_nonfinite_fused(cuda):
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy.uniform([33, 33, 33])
    x = torch.rand(33, 33, 33, dtype=torch.float64, device=cuda)
    x[17, 5, 30] = float("inf")
    with pytest.raises(hgr.HgrError, match="non-finite"):
        hgr.decompose(x, g)
    plan = hgr.Plan(g, "f64")
    plan.decompose_(x)
    with pytest.raises(hgr.HgrError, match="non-finite"):
        plan.sync_status()


@pytest.mark.parametrize("shape", [(33, 17, 9), (65, 129), (257,)], ids=str)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_device_synthetic_field_bitwise(cuda, shape, dt):
    """bench.py's device field == tests/synthetic.smooth_field, bit for bit."""
    hgr = _hgr()
    from tests.synthetic import smooth_field
    dev = hgr.synthetic_field(shape, dt, seed=12345, device=cuda).cpu().numpy()
    host = smooth_field(shape, np.float64 if dt == "f64" else np.float32, 12345)
    assert np.array_equal(dev, host)


@pytest.mark.parametrize("shape", [(65, 65, 65), (129, 65, 33)], ids=str)
def test_profiled_run_matches_unprofiled(cuda, shape):
    """The per-launch event profile (bench roofline) does not change results."""
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy.uniform(list(shape))
    x = hgr.synthetic_field(shape, "f64", device=cuda)
    plan = hgr.Plan(g, "f64")
    a, b = torch.empty_like(x), torch.empty_like(x)
    plan.decompose_into(x, a)
    plan.set_profiling(True)
    plan.decompose_into(x, b)
    prof = plan.read_profile()
    plan.set_profiling(False)
    assert torch.equal(a, b)
    assert prof["fused_decompose_level"][2] >= 1 and prof["thomas"][2] >= 3
