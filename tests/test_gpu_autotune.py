"""Tile-segment autotuning (reference perf_model.hpp:71-137).

The plan ranks each fused kernel's segment lengths with the sector model,
times the top three and keeps the fastest. Segmenting only changes which CTA
computes a coarse plane, never the arithmetic, so tuned results must be
bit-identical to the heuristic's; both must match the reference.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,dt", [((257, 257, 257), "f32"), ((129, 257, 129), "f64")],
                         ids=["257^3_f32", "129x257x129_f64"])
def test_autotune_report_and_bitwise_results(cuda, shape, dt):
    import torch
    import paper_2007_04457_b200 as hgr
    from tests.synthetic import smooth_field
    g = hgr.GridHierarchy.uniform(list(shape))
    L = g.levels()
    plan = hgr.Plan(g, dt)
    npdt = np.float64 if dt == "f64" else np.float32
    u = smooth_field(shape, npdt, 4242)
    x = torch.from_numpy(u).to(cuda)

    p0, y0 = torch.empty_like(x), torch.empty_like(x)
    plan.decompose_into(x, p0)
    plan.recompose_into(p0, y0, L)

    scratch = torch.empty_like(x)
    rep = plan.autotune(x, scratch)
    entries = rep["kernels"]
    kinds = {(e["level"], e["kernel"]) for e in entries}
    big = [l for l in range(1, L + 1) if g.level_node_count(l) >= (1 << 15)]
    for l in big:
        for k in ("decompose_level", "recompose_level", "recompose_interp"):
            assert (l, k) in kinds, (l, k)
    for e in entries:
        c = e["candidates"]
        models = [v["model_us"] for v in c]
        assert models == sorted(models), "candidates ranked by the model"
        timed = [v for v in c if v["measured_us"] is not None]
        assert len(timed) == min(3, len(c)), "the top three are measured"
        assert all(v["measured_us"] is None for v in c[len(timed):])
        best = min(timed, key=lambda v: v["measured_us"])
        assert e["chosen_s0"] == best["s0"]

    p1, y1 = torch.empty_like(x), torch.empty_like(x)
    plan.decompose_into(x, p1)
    plan.recompose_into(p1, y1, L)
    assert torch.equal(p0, p1), "tuned decompose differs from the heuristic's"
    assert torch.equal(y0, y1), "tuned recompose differs from the heuristic's"

    O = oracle.Oracle("reference" if oracle.available("reference") else "port")
    expect = O.decompose(u)
    tol = 1e-12 if dt == "f64" else 1e-5
    err = float(np.abs(p1.cpu().numpy().astype(np.float64) - expect).max()) / float(np.abs(u).max())
    assert err <= tol

    plan.reset_tuning()
    p2 = torch.empty_like(x)
    plan.decompose_into(x, p2)
    assert torch.equal(p0, p2)


def test_env_autotune_first_decompose(cuda):
    """HGR_AUTOTUNE=1: the first out-of-place decompose tunes the plan first and
    still returns the right pyramid (bit-identical to an untuned plan)."""
    import os
    import torch
    import paper_2007_04457_b200 as hgr
    shape = [129, 129, 257]
    g = hgr.GridHierarchy.uniform(shape)
    x = hgr.synthetic_field(shape, "f32", seed=11, device=cuda)
    ref = torch.empty_like(x)
    hgr.Plan(g, "f32").decompose_into(x, ref)
    old = os.environ.get("HGR_AUTOTUNE")
    os.environ["HGR_AUTOTUNE"] = "1"
    try:
        plan = hgr.Plan(g, "f32")
    finally:
        if old is None:
            del os.environ["HGR_AUTOTUNE"]
        else:
            os.environ["HGR_AUTOTUNE"] = old
    out = torch.empty_like(x)
    plan.decompose_into(x, out)
    plan.sync_status()
    assert torch.equal(out, ref)
