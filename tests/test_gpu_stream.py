"""GPU parity of the streaming IPK passes (csrc/kernels_stream.cu): the Thomas
passes of 3D levels (thomas_pass, correction.hpp:262-278) as column solves
streamed band by band through a shared-memory ring -- dim 0 as column strips of
the c0 x (c1*c2) matrix; fp32 dims 1+2 on whole planes (rows along dim 2, then
columns along dim 1); fp64 dim-1 strips of every plane plus the row kernel.

The shapes give coarse extents with lines shorter than one band, lines that are
not a multiple of the band length (16), strips of one and several jobs per
matrix, plane rows of every row-chunk class (c2 <= 160, <= 288, <= 544),
non-uniform coordinates and a level with more planes than SMs. Every
decompose / recompose is compared with the oracle at north_star's tolerance and
with the plan's other IPK path (HGR_THOMAS_STREAM=0) of the same build.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _stream_every_level(monkeypatch):
    # fp64 levels under 2^20 coarse nodes take the three-pass kernels by default
    # (plan.cu stream_min_); these shapes are small so that they cover the
    # streaming passes, so switch the threshold off
    monkeypatch.setenv("HGR_STREAM_MIN", "0")


def _hgr():
    import paper_2007_04457_b200 as hgr
    return hgr


def _nonuniform(shape, seed=0):
    return [oracle.random_coords(n, 7001 + seed + d) for d, n in enumerate(shape)]


CASES = [
    ((129, 129, 129), np.float64, False),   # coarse 65^3: 5 bands, K clamped to 4
    ((257, 129, 65), np.float32, True),     # coarse 129x65x33: plane rows c2 = 33
    ((65, 513, 129), np.float64, True),     # coarse 33x257x65
    ((257, 257, 257), np.float32, False),   # coarse 129^3
    ((129, 257, 1025), np.float64, False),  # coarse 65x129x513: dim-1 strips of 2 jobs
    ((513, 65, 257), np.float64, True),     # coarse 257x33x129: 257 lines of dim 0
    ((33, 1025, 513), np.float32, True),    # coarse 17x513x257: plane rows c2 = 257
    ((1025, 33, 33), np.float32, False),    # coarse 513x17x17: narrow strips
    ((17, 65, 1025), np.float32, False),    # coarse 9x33x513: dim-0 lines of 9 (1 band)
    ((33, 33, 1025), np.float64, True),     # coarse 17x17x513: two bands of 16 + 1
]


def _ids(c):
    return "x".join(map(str, c[0])) + ("_f64" if c[1] == np.float64 else "_f32") + \
        ("_nu" if c[2] else "")


# lookahead forced up (HGR_STREAM_K): fp32 levels whose uniform spacings need one
# lookahead band otherwise take the shared-memory path of the pending bands
FORCED_K = [((257, 257, 257), np.float32, False), ((33, 1025, 513), np.float32, True),
            ((129, 129, 129), np.float64, False)]


@pytest.mark.parametrize("shape,dt,nonuniform", FORCED_K, ids=[_ids(c) for c in FORCED_K])
@pytest.mark.parametrize("k", ["2", "4"])
def test_stream_thomas_forced_lookahead(cuda, port, parity_log, monkeypatch, shape, dt,
                                        nonuniform, k):
    monkeypatch.setenv("HGR_STREAM_K", k)
    test_stream_thomas_vs_oracle(cuda, port, parity_log, monkeypatch, shape, dt, nonuniform)


# two pending bands in registers (HGR_STREAM_KR=2: read once per process, so in
# a child process)
@pytest.mark.parametrize("shape", ["17x257x129", "129x129x129"])
def test_stream_two_register_bands(cuda, shape):
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, HGR_STREAM_KR="2", CFG=shape)
    out = subprocess.run([sys.executable, str(root / "tools" / "dbg_inplace.py"), shape, "f64"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = out.stdout.strip().splitlines()[-1]
    err = float(line.split("out-of-place err")[1].split()[0])
    assert err <= 1e-12 * 1.5, line  # dbg_inplace reports max-abs error (|u| <= 1.5)
    import re
    nans = re.findall(r"np\.int64\((\d+)\)", line)
    assert nans and all(v == "0" for v in nans), line  # no NaN from the in-place runs


# fp64 whole-plane pass with the pending bands corrected in place (off by default)
PLANES64 = [c for c in CASES if c[1] == np.float64]


@pytest.mark.parametrize("shape,dt,nonuniform", PLANES64, ids=[_ids(c) for c in PLANES64])
def test_stream_planes64_vs_oracle(cuda, port, parity_log, monkeypatch, shape, dt, nonuniform):
    monkeypatch.setenv("HGR_STREAM_PLANES64", "1")
    test_stream_thomas_vs_oracle(cuda, port, parity_log, monkeypatch, shape, dt, nonuniform)


@pytest.mark.parametrize("shape,dt,nonuniform", CASES, ids=[_ids(c) for c in CASES])
def test_stream_thomas_vs_oracle(cuda, port, parity_log, monkeypatch, shape, dt, nonuniform):
    import torch
    hgr = _hgr()
    coords = _nonuniform(shape) if nonuniform else None
    g = hgr.GridHierarchy(coords) if coords else hgr.GridHierarchy.uniform(list(shape))
    rng = np.random.default_rng(13)
    u = rng.uniform(-1, 1, shape).astype(dt)
    scale = float(np.abs(u).max())
    tol = 1e-12 if dt == np.float64 else 1e-5
    tag = "f64" if dt == np.float64 else "f32"
    want = port.decompose(u, coords)
    want64 = want.astype(np.float64)
    x = torch.from_numpy(u).to(cuda)
    outs = {}
    for stream in ("1", "0"):
        monkeypatch.setenv("HGR_THOMAS_STREAM", stream)
        plan = hgr.Plan(g, tag)
        p = torch.empty_like(x)
        plan.decompose_into(x, p)
        plan.sync_status()
        y = torch.empty_like(x)
        plan.recompose_into(p, y, g.levels())
        r = torch.empty_like(x)
        plan.recompose_into(torch.from_numpy(want).to(cuda), r, g.levels())
        outs[stream] = (p.cpu().numpy().astype(np.float64), y, r.cpu().numpy().astype(np.float64))
    p1, y1, r1 = outs["1"]
    p0, _, r0 = outs["0"]
    rec_want = port.recompose(want, g.levels(), coords).astype(np.float64)
    errs = {
        "decompose_vs_oracle": float(np.abs(p1 - want64).max()) / scale,
        "recompose_vs_oracle": float(np.abs(r1 - rec_want).max()) / scale,
        "round_trip": float((y1.double() - x.double()).abs().max().item()) / scale,
        "stream_vs_other_decompose": float(np.abs(p1 - p0).max()) / scale,
        "stream_vs_other_recompose": float(np.abs(r1 - r0).max()) / scale,
    }
    parity_log(f"stream_{_ids((shape, dt, nonuniform))}", **errs)
    for k, v in errs.items():
        assert v <= tol, f"{k}: {v:.3e} > {tol}"
