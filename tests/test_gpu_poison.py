"""Read-before-write guard: plans whose workspace is NaN-filled at creation
(HGR_POISON_WORKSPACE=1) must give the same results. Any kernel that reads a
workspace value it did not write first -- including padding beyond an array
that is multiplied by a zero table entry (NaN * 0 = NaN) -- shows up as a
non-finite or wrong output here."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SHAPES = [((9, 129, 33), "f32"), ((9, 129, 33), "f64"), ((65, 65, 65), "f32"),
          ((33, 17, 9), "f64"), ((129, 33, 17), "f32"), ((5, 65, 257), "f64"),
          ((257, 257), "f32"), ((513, 513), "f64"), ((4097, 65), "f32"),
          ((65537,), "f32"), (((1 << 20) + 1,), "f64"), ((17,), "f64"), ((3, 3), "f32")]


@pytest.fixture
def poisoned():
    old = os.environ.get("HGR_POISON_WORKSPACE")
    os.environ["HGR_POISON_WORKSPACE"] = "1"
    yield
    if old is None:
        del os.environ["HGR_POISON_WORKSPACE"]
    else:
        os.environ["HGR_POISON_WORKSPACE"] = old


@pytest.mark.parametrize("shape,dt", SHAPES, ids=["x".join(map(str, s)) + "_" + d for s, d in SHAPES])
def test_poisoned_workspace(cuda, poisoned, shape, dt):
    import torch
    import paper_2007_04457_b200 as hgr
    from tests.synthetic import smooth_field
    npdt = np.float64 if dt == "f64" else np.float32
    g = hgr.GridHierarchy.uniform(list(shape))
    L = g.levels()
    u = smooth_field(shape, npdt, 99)
    scale = float(np.abs(u).max())
    tol = 1e-12 if dt == "f64" else 1e-5
    plan = hgr.Plan(g, dt)
    x = torch.from_numpy(u).to(cuda)
    p = torch.empty_like(x)
    plan.decompose_into(x, p)
    plan.sync_status()
    O = oracle.Oracle("reference" if oracle.available("reference") else "port")
    expect = O.decompose(u)
    got = p.cpu().numpy().astype(np.float64)
    assert np.isfinite(got).all()
    assert float(np.abs(got - expect).max()) / scale <= tol
    for m in sorted({L, max(0, L - 1), 0}):
        y = torch.empty_like(x)
        plan.recompose_into(p, y, m)
        want = O.recompose(expect.astype(npdt), m)
        err = float(np.abs(y.cpu().numpy().astype(np.float64) - want).max()) / scale
        assert err <= tol, (m, err)
    q = x.clone()
    plan.decompose_(q)
    plan.sync_status()
    assert float((q.double() - p.double()).abs().max()) / scale <= tol
