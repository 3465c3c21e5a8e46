"""The drop-in boundary's contract on the GPU: concurrency
("distinct arrays may be processed concurrently" -- threads and
streams on one grid give the serial results bitwise), operands the TMA kernels
cannot take (16-byte misaligned views take the reference path and still match
the oracle), argument validation of the plan API, the host-pointer path
(pageable and pinned) equal to the device path, and the device error report,
transfer and apply_coefficients against the oracle."""
import threading

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _hgr():
    import paper_2007_04457_b200 as hgr
    return hgr


def _field(shape, dt, seed):
    return np.random.default_rng(seed).uniform(-1, 1, shape).astype(dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_concurrent_streams_one_grid_bitwise(cuda, dt):
    """Four host threads, each on its own CUDA stream, decompose + recompose
    different arrays of the same (fused-size) grid through the one-shot C ABI,
    three times over; every result equals the serial one bitwise."""
    import torch
    hgr = _hgr()
    shape = (65, 65, 129)
    g = hgr.GridHierarchy.uniform(list(shape))
    ins = [torch.from_numpy(_field(shape, dt, 40 + t)).to(cuda) for t in range(4)]
    serial = []
    for x in ins:
        r = hgr.decompose(x, g)
        serial.append((r.data.clone(), hgr.recompose(r, g.levels()).clone()))
    torch.cuda.synchronize()
    errors = []

    def work(t, out):
        try:
            with torch.cuda.stream(torch.cuda.Stream(cuda)):
                for _ in range(3):
                    r = hgr.decompose(ins[t], g)
                    back = hgr.recompose(r, g.levels())
                    torch.cuda.current_stream().synchronize()
                    out.append((r.data, back))
        except Exception as e:  # surfaced below
            errors.append(e)

    outs = [[] for _ in ins]
    th = [threading.Thread(target=work, args=(t, outs[t])) for t in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    for t in range(4):
        for pyr, back in outs[t]:
            assert torch.equal(pyr, serial[t][0])
            assert torch.equal(back, serial[t][1])


def test_concurrent_host_calls_bitwise(cuda):
    """The host-pointer entry points (the C++ templates' path) from several
    threads at once: the plan pool gives each its own workspace."""
    hgr = _hgr()
    shape = (33, 65, 65)
    g = hgr.GridHierarchy.uniform(list(shape))
    ins = [_field(shape, np.float64, 60 + t) for t in range(4)]
    serial = [hgr.decompose(u, g).data for u in ins]
    res = [None] * 4

    def work(t):
        res[t] = [hgr.decompose(ins[t], g).data for _ in range(3)]

    th = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for t in range(4):
        for a in res[t]:
            assert np.array_equal(a, serial[t])


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("shape", [(65, 65, 65), (257, 129), (4097,)], ids=lambda s: "x".join(map(str, s)))
def test_misaligned_operands(cuda, port, shape, dt):
    """A contiguous view at an odd element offset is not 16-byte aligned: the
    fused TMA kernels reject it and the level takes the reference path (its
    stage buffers are sized for fused-size levels too). Results match the oracle."""
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy.uniform(list(shape))
    u = _field(shape, dt, 7)
    n = u.size
    tol = 1e-12 if dt == np.float64 else 1e-5
    base = torch.empty(n + 1, dtype=torch.float64 if dt == np.float64 else torch.float32, device=cuda)
    view = base[1:].view(shape)
    view.copy_(torch.from_numpy(u))
    assert view.data_ptr() % 16 != 0
    expect = port.decompose(u)
    scale = float(np.abs(u).max())
    plan = hgr.Plan(g, "f64" if dt == np.float64 else "f32")
    obase = torch.empty_like(base)
    out = obase[1:].view(shape)
    for _ in range(2):  # direct launch, then the captured graph
        plan.decompose_into(view, out)
        plan.sync_status()
        got = out.cpu().numpy()
        assert np.abs(got.astype(np.float64) - expect).max() / scale <= tol
    back_base = torch.empty_like(base)
    back = back_base[1:].view(shape)
    for _ in range(2):
        plan.recompose_into(out, back, g.levels())
        torch.cuda.synchronize()
        assert np.abs(back.cpu().numpy().astype(np.float64) - u).max() / scale <= tol
    # one-shot in-place entry point on the misaligned view
    r2 = view.clone()
    hgr._check(getattr(hgr._lib.load(), f"hgr_cuda_decompose_{'f64' if dt == np.float64 else 'f32'}")(
        hgr.C.byref(g.desc), view.data_ptr(), None))
    assert np.abs(view.cpu().numpy().astype(np.float64) - expect).max() / scale <= tol
    del r2


def test_plan_rejects_bad_operands(cuda):
    import torch
    hgr = _hgr()
    g = hgr.GridHierarchy.uniform([17, 17, 17])
    plan = hgr.Plan(g, "f64")
    ok = torch.zeros(17, 17, 17, dtype=torch.float64, device=cuda)
    bad = {
        "dtype": torch.zeros(17, 17, 17, dtype=torch.float32, device=cuda),
        "shape": torch.zeros(17, 17, 9, dtype=torch.float64, device=cuda),
        "contiguous": torch.zeros(17, 17, 34, dtype=torch.float64, device=cuda)[:, :, ::2],
        "CUDA": torch.zeros(17, 17, 17, dtype=torch.float64),
    }
    for what, x in bad.items():
        with pytest.raises(hgr.HgrError, match=what):
            plan.decompose_into(x, ok)
        with pytest.raises(hgr.HgrError, match=what):
            plan.recompose_into(ok, x, 1)
    with pytest.raises(hgr.HgrError):
        hgr.Plan(g, "f16")


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_host_path_equals_device_path(cuda, dt):
    """numpy (pageable, staged through the pinned ring in several chunks) and
    pinned torch host tensors (direct DMA) give the device path's results bitwise."""
    import torch
    hgr = _hgr()
    shape = (129, 257, 257) if dt == np.float32 else (129, 129, 257)  # > 3 staging slots
    g = hgr.GridHierarchy.uniform(list(shape))
    u = _field(shape, dt, 11)
    dev = hgr.decompose(torch.from_numpy(u).to(cuda), g).data.cpu().numpy()
    host = hgr.decompose(u, g).data
    assert np.array_equal(host, dev)
    pinned = torch.from_numpy(u).pin_memory()
    pr = hgr.decompose(pinned, g)
    assert pr.data.is_pinned() and np.array_equal(pr.data.numpy(), dev)
    for m in (g.levels(), 2):
        want = hgr.recompose(hgr.RefactoredArray(torch.from_numpy(dev).to(cuda), g), m).cpu().numpy()
        assert np.array_equal(hgr.recompose(hgr.RefactoredArray(host, g), m), want)
        assert np.array_equal(hgr.recompose(pr, m).numpy(), want)


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_error_report_device(cuda, dt):
    """error_report (refactor.hpp:100-120) as a device reduction vs the
    definition in double; deterministic run to run."""
    import torch
    hgr = _hgr()
    a = _field((33, 65, 129), dt, 3)
    b = (a + _field(a.shape, dt, 4) * 1e-3).astype(dt)
    ad, bd = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d = ad - bd
    want = (np.sqrt((d * d).sum()), np.sqrt((d * d).sum()) / np.sqrt((ad * ad).sum()),
            np.abs(d).max(), np.abs(d).max() / np.abs(ad).max())
    r1 = hgr.error_report(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda))
    r2 = hgr.error_report(a, b)
    got = (r1.l2_abs, r1.l2_rel, r1.linf_abs, r1.linf_rel)
    assert np.allclose(got, want, rtol=1e-12, atol=0)
    assert got == (r2.l2_abs, r2.l2_rel, r2.linf_abs, r2.linf_rel)
    z = np.zeros(8, dt)
    rz = hgr.error_report(z, z + 1)
    assert rz.l2_rel == float("inf") and rz.linf_rel == float("inf") and rz.linf_abs == 1.0
    r0 = hgr.error_report(z, z)
    assert (r0.l2_abs, r0.l2_rel, r0.linf_abs, r0.linf_rel) == (0.0, 0.0, 0.0, 0.0)


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_transfer_and_mass_vs_oracle(cuda, port, dt):
    """transfer_apply (correction.hpp:67-88) and mass_apply on batches of
    non-uniform fibers vs the oracle."""
    hgr = _hgr()
    for n in (3, 5, 33, 1025):
        h = np.diff(oracle.random_coords(n, 5 + n)).astype(dt)
        v = _field((7, n), dt, n)
        got_t = hgr.transfer_apply(v, h)
        got_m = hgr.mass_apply(v, h)
        tol = 1e-14 if dt == np.float64 else 1e-6
        for f in range(7):
            want_t = port.transfer_apply(v[f], h)
            want_m = port.mass_apply(v[f], h)
            assert np.abs(got_t[f] - want_t).max() <= tol * max(1.0, np.abs(want_t).max())
            assert np.abs(got_m[f] - want_m).max() <= tol * max(1.0, np.abs(want_m).max())
    with pytest.raises(hgr.HgrError, match="odd"):
        hgr.transfer_apply(np.zeros(4, dt), np.ones(3, dt))


@pytest.mark.parametrize("shape", [(9, 17, 33), (65, 65), (129,)], ids=lambda s: "x".join(map(str, s)))
def test_apply_coefficients_vs_oracle(cuda, port, shape):
    hgr = _hgr()
    coords = [oracle.random_coords(n, 30 + d) for d, n in enumerate(shape)]
    g = hgr.GridHierarchy(coords)
    L = g.levels()
    coarse = _field(tuple(g.level_extents(L - 1)), np.float64, 1)
    coeffs = _field(tuple(g.level_extents(L)), np.float64, 2)
    want = port.interpolate_to_fine(coarse, shape, L, coords) + coeffs
    got = hgr.apply_coefficients(coarse, coeffs, g, L)
    assert np.abs(got - want).max() <= 1e-14


@pytest.mark.parametrize("shape", [(2097153,), (33, 65, 129)], ids=["1d_2M", "3d"])
def test_plan_cache_keys_by_coordinates(cuda, port, shape):
    """The one-shot calls' plan cache keys a grid by its coordinates, compared in
    place (chunked over host threads for long 1D grids): a uniform grid, a
    non-uniform one and a copy of it with one coordinate moved share extents but
    never a plan; each call matches the oracle on its own grid."""
    hgr = _hgr()
    c1 = [oracle.random_coords(n, 900 + d) for d, n in enumerate(shape)]
    c2 = [c.copy() for c in c1]
    last = c2[-1]
    k = len(last) // 2 + 1
    last[k] = 0.5 * (last[k] + last[k + 1])  # still strictly increasing
    grids = {"uniform": (hgr.GridHierarchy.uniform(list(shape)), None),
             "c1": (hgr.GridHierarchy(c1), c1), "c2": (hgr.GridHierarchy(c2), c2)}
    u = _field(shape, np.float64, 5)
    scale = float(np.abs(u).max())
    for name in ("uniform", "c1", "c2", "uniform", "c2", "c1"):
        g, coords = grids[name]
        got = hgr.decompose(u.copy(), g).data
        want = port.decompose(u, coords)
        assert np.abs(got - want).max() / scale <= 1e-12, name
