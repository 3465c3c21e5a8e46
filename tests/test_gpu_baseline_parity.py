"""Oracle parity at the two 1025^3 BASELINE configurations (SURVEY §8e:
"full oracle parity on rank 0's block"): configs[2] 1025^3 fp64 (the north-star
roofline run) and configs[4] 1025^3 fp32 (the headline weak-scaling block),
against the reference itself (oracle/_ref/libhgr_ref.so, the unmodified
reference headers, run on this box's host cores).

Compared at north_star's tolerance (max-abs / max|u| <= 1e-12 fp64, 1e-5 fp32):
* the decompose pyramid against the reference's (out of place and through the
  in-place entry point),
* the full recompose of the reference's pyramid against the reference's,
* a prefix recompose (classes 0..L-2) against the reference's,
* the GPU round trip against the input.
fp32 additionally: the GPU's fp32 pyramid is within 10x of the reference's own
fp32-vs-fp64 error (both against the reference in fp64 on the same input).
Every measured error is logged (parity_log). Comparisons run on the device.
"""
import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SHAPE = (1025, 1025, 1025)


def _hgr():
    import paper_2007_04457_b200 as hgr
    return hgr


@pytest.fixture(scope="module")
def ref():
    if not oracle.available("reference"):
        pytest.fail("oracle/_ref/libhgr_ref.so missing: build with __graft_entry__.build() "
                    "where /root/reference exists (the library travels with the repo)")
    import os
    os.environ.setdefault("HGR_THREADS", str(len(os.sched_getaffinity(0))))
    O = oracle.Oracle("reference")
    O.set_worker_count(len(os.sched_getaffinity(0)))
    return O


def _rel(a_dev, b_dev, scale):
    return float((a_dev - b_dev).abs().max().item()) / scale


def _run(cuda, ref, parity_log, dt):
    import torch
    hgr = _hgr()
    tag = "f64" if dt == np.float64 else "f32"
    g = hgr.GridHierarchy.uniform(list(SHAPE))
    L = g.levels()
    plan = hgr.Plan(g, tag)
    u = hgr.synthetic_field(SHAPE, tag, seed=12345, device=cuda)  # == tests/synthetic bitwise
    scale = float(u.abs().max().item())
    uh = u.cpu().numpy()
    errs = {}
    ref_p = ref.decompose(uh)
    ref_p_dev = torch.from_numpy(ref_p).to(cuda)
    gpu_p = torch.empty_like(u)
    plan.decompose_into(u, gpu_p)
    plan.sync_status()
    errs["decompose"] = _rel(gpu_p, ref_p_dev, scale)
    # the in-place entry point (hgr_cuda_decompose_* / Plan.decompose_): its own
    # schedule (load-only level kernel + in-place coefficients), same result
    inplace = u.clone()
    plan.decompose_(inplace)
    plan.sync_status()
    errs["decompose_in_place"] = _rel(inplace, ref_p_dev, scale)
    del inplace
    back = torch.empty_like(u)
    plan.recompose_into(gpu_p, back, L)
    errs["round_trip"] = _rel(back, u, scale)
    for m in (L, L - 2):
        want = torch.from_numpy(ref.recompose(ref_p, m)).to(cuda)
        plan.recompose_into(ref_p_dev, back, m)
        errs[f"recompose_upto_{m}"] = _rel(back, want, scale)
        del want
    if dt == np.float32:
        # the reference in fp64 on the same (fp32-valued) input: how far each fp32
        # pyramid is from the fp64 one
        p64 = torch.from_numpy(ref.decompose(uh.astype(np.float64))).to(cuda)
        errs["gpu_f32_vs_ref_f64"] = _rel(gpu_p.double(), p64, scale)
        errs["ref_f32_vs_ref_f64"] = _rel(ref_p_dev.double(), p64, scale)
        del p64
    del ref_p, ref_p_dev, gpu_p, back, u
    torch.cuda.empty_cache()
    parity_log(f"1025^3_{tag}_vs_reference", shape=list(SHAPE), levels=L, **errs)
    return errs


def test_1025_f64_vs_reference(cuda, ref, parity_log):
    errs = _run(cuda, ref, parity_log, np.float64)
    for k, v in errs.items():
        assert v <= 1e-12, f"{k}: {v:.3e}"


def test_1025_f32_vs_reference(cuda, ref, parity_log):
    errs = _run(cuda, ref, parity_log, np.float32)
    for k in ("decompose", "decompose_in_place", "round_trip", "recompose_upto_10",
              "recompose_upto_8"):
        assert errs[k] <= 1e-5, f"{k}: {errs[k]:.3e}"
    assert errs["gpu_f32_vs_ref_f64"] <= 10 * errs["ref_f32_vs_ref_f64"], errs
