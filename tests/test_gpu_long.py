"""GPU parity on grids whose Thomas lines exceed one register tile.

Rows longer than the row tiles take k_thomas_long, strided lines longer than
16 chunks take the windowed k_thomas_lines; lines longer than one window are
cut into overlapping windows whose outside carry is dropped (below 2^-56 /
2^-26 of it, kernels_thomas.cu), and those passes run out of place through the
plan's scratch buffer. Compared with the reference (oracle/_ref) on decompose,
recompose of the reference pyramid, a prefix recompose, and the in-place
decompose entry point. Tolerances are north_star's: 1e-12*max|u| (fp64),
1e-5*max|u| (fp32).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _nonuniform(shape):
    return [np.expm1(2.0 * np.arange(n) / (n - 1)) / np.expm1(2.0) for n in shape]


CASES = [
    # 2D: windowed strided lines (2049) and windowed rows (4097 > one fp64 window)
    ((4097, 8193), np.float64, True),
    # 2D fp32: windowed strided lines (4097), long rows in one window (2049)
    ((8193, 4097), np.float32, False),
    # 1D: one row of 2^21+1 coarse nodes, hundreds of windows
    (((1 << 22) + 1,), np.float64, True),
    (((1 << 21) + 1,), np.float32, False),
    # 3D: windowed strided lines along dim 1 (1025 coarse), short dims around it
    ((33, 2049, 65), np.float64, True),
    ((65, 17, 4097), np.float32, True),
]


@pytest.mark.parametrize("shape,dt,nonuniform", CASES,
                         ids=["x".join(map(str, c[0])) + ("_f64" if c[1] == np.float64 else "_f32")
                              for c in CASES])
def test_long_lines_vs_reference(cuda, shape, dt, nonuniform):
    import torch
    import paper_2007_04457_b200 as hgr
    from tests.synthetic import smooth_field
    coords = _nonuniform(shape) if nonuniform else None
    g = hgr.GridHierarchy(coords) if coords else hgr.GridHierarchy.uniform(list(shape))
    L = g.levels()
    u = smooth_field(shape, dt, 777)
    scale = float(np.abs(u).max())
    tol = 1e-12 if dt == np.float64 else 1e-5
    O = oracle.Oracle("reference" if oracle.available("reference") else "port")
    expect = O.decompose(u, coords)
    plan = hgr.Plan(g, "f64" if dt == np.float64 else "f32")
    x = torch.from_numpy(u).to(cuda)
    p = torch.empty_like(x)
    plan.decompose_into(x, p)
    plan.sync_status()
    err = float(np.abs(p.cpu().numpy().astype(np.float64) - expect).max()) / scale
    assert err <= tol, f"decompose vs {O.kind}: {err:.3e}"

    # in-place entry point
    q = x.clone()
    plan.decompose_(q)
    plan.sync_status()
    err_ip = float((q.double() - p.double()).abs().max().item()) / scale
    assert err_ip <= tol, f"in-place decompose: {err_ip:.3e}"

    # recompose of the reference's own pyramid
    ref_p = torch.from_numpy(expect.astype(dt)).to(cuda)
    y = torch.empty_like(x)
    plan.recompose_into(ref_p, y, L)
    err_r = float((y.double() - x.double()).abs().max().item()) / scale
    assert err_r <= tol, f"recompose(reference pyramid): {err_r:.3e}"

    # prefix recompose against the reference's prefix recompose
    m = max(0, L - 2)
    want = O.recompose(expect, m, coords)
    plan.recompose_into(ref_p, y, m)
    err_m = float(np.abs(y.cpu().numpy().astype(np.float64) - want).max()) / scale
    assert err_m <= tol, f"recompose(upto {m}) vs {O.kind}: {err_m:.3e}"


@pytest.mark.parametrize("shape,dt,limit_ms", [(((1 << 24) + 1,), "f64", 25.0),
                                                ((4097, 4097), "f32", 15.0),
                                                ((129, 129, 4097), "f32", 25.0)],
                         ids=["line_2^24+1_f64", "4097^2_f32", "129x129x4097_f32"])
def test_long_shapes_time_bound(cuda, shape, dt, limit_ms):
    """Guard against a serial fallback on long lines (a warp or a thread per
    line of millions of nodes): loose bounds, ~10x above the measured times."""
    import torch
    import paper_2007_04457_b200 as hgr
    g = hgr.GridHierarchy.uniform(list(shape))
    plan = hgr.Plan(g, dt)
    x = hgr.synthetic_field(list(shape), dt, seed=5, device=cuda)
    p, y = torch.empty_like(x), torch.empty_like(x)
    for _ in range(2):
        plan.decompose_into(x, p)
        plan.recompose_into(p, y, g.levels())
    torch.cuda.synchronize(cuda)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    plan.decompose_into(x, p)
    plan.recompose_into(p, y, g.levels())
    ev1.record()
    torch.cuda.synchronize(cuda)
    ms = ev0.elapsed_time(ev1)
    assert ms < limit_ms, f"round trip {ms:.2f} ms"
