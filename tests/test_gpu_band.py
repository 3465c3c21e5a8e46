"""GPU parity of the cluster IPK path (csrc/kernels_band.cu): 3D levels solve
their Thomas passes (thomas_pass, correction.hpp:262-278) as a dim-0 band pass
plus a fused dims-1+2 plane pass, lines cut into bands of <= 33 positions, one
CTA each, carries exchanged through distributed shared memory.

Shapes are chosen so the coarse extents give clusters of 1, 2, 4, 8 and 16
bands, unequal bands (n not a multiple of the band count), rows of every
row-tile class (c2 = 33, 65, 129, 257, 513) and non-uniform coordinates.
Each decompose / recompose is compared with the oracle at north_star's
tolerance, for both dim-0 strategies (HGR_THOMAS_BAND=1: strided-line dim 0;
=2: cluster band pass for dim 0 too), and with the three-pass path
(HGR_THOMAS_BAND=0) of the same build. The streaming passes that precede the
band kernels in the plan are switched off here (HGR_THOMAS_STREAM=0).
"""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _no_stream(monkeypatch):
    monkeypatch.setenv("HGR_THOMAS_STREAM", "0")


def _hgr():
    import paper_2007_04457_b200 as hgr
    return hgr


def _nonuniform(shape, seed=0):
    return [oracle.random_coords(n, 9001 + seed + d) for d, n in enumerate(shape)]


CASES = [
    ((129, 129, 129), np.float64, False),   # coarse 65^3: 2 bands
    ((257, 129, 65), np.float32, True),     # coarse 129x65x33: 4 / 2 bands, c2 = 33
    ((65, 513, 129), np.float64, True),     # coarse 33x257x65: 1 / 8 bands
    ((257, 257, 257), np.float32, False),   # coarse 129^3: 4 bands, c2 = 129
    ((129, 257, 1025), np.float64, False),  # coarse 65x129x513: c2 = 513
    ((513, 65, 257), np.float64, True),     # coarse 257x33x129: 8 / 1 bands
]


@pytest.mark.parametrize("shape,dt,nonuniform", CASES,
                         ids=["x".join(map(str, c[0])) + ("_f64" if c[1] == np.float64 else "_f32")
                              + ("_nu" if c[2] else "") for c in CASES])
def test_band_thomas_vs_oracle(cuda, port, parity_log, shape, dt, nonuniform):
    import torch
    hgr = _hgr()
    coords = _nonuniform(shape) if nonuniform else None
    g = hgr.GridHierarchy(coords) if coords else hgr.GridHierarchy.uniform(list(shape))
    rng = np.random.default_rng(11)
    u = rng.uniform(-1, 1, shape).astype(dt)
    scale = float(np.abs(u).max())
    tol = 1e-12 if dt == np.float64 else 1e-5
    tag = "f64" if dt == np.float64 else "f32"
    want = port.decompose(u, coords)
    want64 = want.astype(np.float64)
    x = torch.from_numpy(u).to(cuda)
    outs = {}
    for band in ("1", "2", "0"):
        os.environ["HGR_THOMAS_BAND"] = band
        try:
            plan = hgr.Plan(g, tag)
        finally:
            os.environ.pop("HGR_THOMAS_BAND", None)
        p = torch.empty_like(x)
        plan.decompose_into(x, p)
        plan.sync_status()
        y = torch.empty_like(x)
        plan.recompose_into(p, y, g.levels())
        outs[band] = (p.cpu().numpy().astype(np.float64), y)
    p1, y1 = outs["1"]
    p2, y2b = outs["2"]
    p0, _ = outs["0"]
    errs = {
        "decompose_vs_oracle": float(np.abs(p1 - want64).max()) / scale,
        "band_all_vs_oracle": float(np.abs(p2 - want64).max()) / scale,
        "band_vs_three_pass": float(np.abs(p1 - p0).max()) / scale,
        "round_trip_band_all": float((y2b.double() - x.double()).abs().max().item()) / scale,
        "round_trip": float((y1.double() - x.double()).abs().max().item()) / scale,
    }
    y2 = torch.empty_like(x)
    os.environ["HGR_THOMAS_BAND"] = "1"
    try:
        plan = hgr.Plan(g, tag)
    finally:
        os.environ.pop("HGR_THOMAS_BAND", None)
    plan.recompose_into(torch.from_numpy(want).to(cuda), y2, g.levels())
    rec_want = port.recompose(want, g.levels(), coords).astype(np.float64)
    errs["recompose_vs_oracle"] = float(np.abs(y2.cpu().numpy().astype(np.float64) - rec_want).max()) / scale
    parity_log(f"band_{'x'.join(map(str, shape))}_{tag}", **errs)
    for k, v in errs.items():
        assert v <= tol, f"{k}: {v:.3e} > {tol}"
