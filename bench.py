#!/usr/bin/env python
"""bench.py -- refactor GB/s (decompose + recompose) on B200, % of HBM roofline.

Metric (BASELINE.json): "refactor GB/s (decompose+recompose) at 1/2/4/8 B200,
% HBM roofline". One step = one full multilevel decompose (out of place) plus
one full recompose (all classes) of a synthetic smooth-plus-noise field on each
GPU; value = sum over GPUs of 2*N*S bytes / step time (max over ranks), i.e.
the paper's round-trip refactoring throughput.

Default workload = BASELINE configs[4], the configuration the 1/2/4/8-GPU
metric is quoted on: an independent 1025^3 fp32 block per GPU (weak scaling).
--config selects the other BASELINE shapes (513^3 fp32, 1025^3 fp64,
257x513x1025 fp64 nonuniform, 513^2 fp64).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME]
  python bench.py --impl reference ...   # the reference's CPU implementation

Launch with torchrun for N > 1 (one process per GPU, NCCL only for the final
max-time / checksum reductions; the blocks are independent).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "weak1025f32": dict(shape=(1025, 1025, 1025), dtype="f32", nonuniform=False,
                        workload="weak scaling: independent 1025^3 fp32 blocks per GPU "
                                 "(BASELINE configs[4])",
                        sample=(513, 513, 513)),
    "513f32": dict(shape=(513, 513, 513), dtype="f32", nonuniform=False,
                   workload="3D 513^3 fp32 uniform grid, all levels (BASELINE configs[1])",
                   sample=(257, 257, 257)),
    "1025f64": dict(shape=(1025, 1025, 1025), dtype="f64", nonuniform=False,
                    workload="3D 1025^3 fp64 uniform grid roofline run (BASELINE configs[2])",
                    sample=(513, 513, 513)),
    "aniso_nu_f64": dict(shape=(257, 513, 1025), dtype="f64", nonuniform=True,
                         workload="3D 257x513x1025 fp64 non-uniform coordinates "
                                  "(BASELINE configs[3])",
                         sample=(65, 129, 257)),
    "513sq_f64": dict(shape=(513, 513), dtype="f64", nonuniform=False,
                      workload="2D 513x513 fp64 uniform grid (BASELINE configs[0])",
                      sample=(513, 513)),
    # not BASELINE configs: large 2D / 1D grids for tuning the 2D / 1D paths
    "8193sq_f32": dict(shape=(8193, 8193), dtype="f32", nonuniform=False,
                       workload="2D 8193x8193 fp32 uniform grid (extra, not in BASELINE)",
                       sample=(1025, 1025)),
    "line_f64": dict(shape=((1 << 26) + 1,), dtype="f64", nonuniform=False,
                     workload="1D 2^26+1 fp64 uniform line (extra, not in BASELINE)",
                     sample=((1 << 20) + 1,)),
}
DEFAULT_CONFIG = "weak1025f32"
# measured beside the default workload in the same run (N = 1): the north-star
# roofline configuration
EXTRA_CONFIGS = ("1025f64",)
FALLBACK_HBM_GBS = 6650.0


def coords_for(shape, nonuniform):
    """Non-uniform coordinates: x_i = (e^{2i/(n-1)} - 1)/(e^2 - 1)."""
    if not nonuniform:
        return None
    return [np.expm1(2.0 * np.arange(n) / (n - 1)) / np.expm1(2.0) for n in shape]


def host_field(shape, dtype, seed):
    from tests.synthetic import smooth_field
    return smooth_field(shape, np.float64 if dtype == "f64" else np.float32, seed)


def algorithmic_bytes(shape, S):
    """Reference-step byte model of SURVEY.md §8(d), per direction."""
    n_d = list(shape)
    D = len(shape)
    L = min((n - 1).bit_length() - 1 for n in n_d)
    total = 0
    for l in range(L, 0, -1):
        s = 1 << (L - l)
        e = [(n - 1) // s + 1 for n in n_d]
        c = [(x - 1) // 2 + 1 for x in e]
        n = int(np.prod(e))
        cn = int(np.prod(c))
        r = n - cn
        stages = [n]
        for k in range(D):
            stages.append(int(np.prod(c[:k + 1] + e[k + 1:])))
        b = (n + r) + (r + stages[1]) + sum(stages[k] + stages[k + 1] for k in range(1, D))
        b += 2 * D * cn + 3 * cn
        total += S * b
    return total


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
                power.append(float(f[7]))
            except ValueError:
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


def shard_seed(rank):
    """Each rank refactors its own independent block: seed 12345 + rank."""
    return 12345 + rank


def reduce_across_ranks(ms_step, checksum, device=None):
    """The only collectives of a multi-GPU run, after the timed region: max of
    the per-rank step time and sum of the per-block checksums.
    Works with NCCL (GPU tensors) or gloo (CPU tensors, tests)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(ms_step)], dtype=torch.float64, device=device)
    c = torch.tensor([float(checksum)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return float(t.item()), float(c.item())


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except (KeyError, ValueError):
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_name, kind):
    """DRAM bytes per launch of the dominant kernel from a committed ncu capture."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(config_name, {}).get(kind)
    except ValueError:
        return None


# ------------------------------------------------------------------------------
# CPU reference arm / CPU baseline (oracle is test infrastructure: used here only
# as the timed baseline, never as the product path)
# ------------------------------------------------------------------------------

def _cpu_oracle():
    """The reference's own CPU implementation for timing: the unmodified headers
    built -O3 -march=native, else the portable build, else the
    C port."""
    import oracle
    for kind in ("reference-native", "reference", "port"):
        if oracle.available(kind):
            return oracle.Oracle(kind), kind
    raise SystemExit("no CPU oracle built (make -C oracle)")


def _describe(kind):
    return {"reference-native": "oracle/_ref/libhgr_ref_native.so: the unmodified reference headers, "
                                "g++ -O3 -march=native",
            "reference": "oracle/_ref/libhgr_ref.so: the unmodified reference headers, g++ -O3",
            "port": "oracle port (C restatement)"}[kind]


def cpu_reference_run(cfg, seconds_budget=None, steps=None, warmup=0, full=False):
    """Round trips (decompose + full recompose) of the reference CPU path on all
    host threads. full=False: the bounded sample cfg["sample"] (the cpu_baseline
    of the GPU line); full=True: the configuration itself (--impl reference),
    warm-up calls on the sample so the timed ones are the workload's."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    os.environ["HGR_THREADS"] = str(cores)
    O, kind = _cpu_oracle()
    O.set_worker_count(cores)
    shape = cfg["shape"] if full else cfg["sample"]
    coords = coords_for(shape, cfg["nonuniform"])
    wshape = cfg["sample"]
    wcoords = coords_for(wshape, cfg["nonuniform"])
    for i in range(warmup):
        uw = host_field(wshape, cfg["dtype"], 12345)
        O.recompose(O.decompose(uw, wcoords), O.levels(wshape, wcoords), wcoords)
    u = host_field(shape, cfg["dtype"], 12345)
    S = u.dtype.itemsize
    L = O.levels(shape, coords)
    times, t_dec, t_rec = [], [], []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        p = O.decompose(u, coords)
        t1 = time.perf_counter()
        back = O.recompose(p, L, coords)
        t2 = time.perf_counter()
        del p
        times.append(t2 - t0)
        t_dec.append(t1 - t0)
        t_rec.append(t2 - t1)
        if steps is not None and len(times) >= steps:
            break
        if seconds_budget is not None and time.perf_counter() - t_start >= seconds_budget:
            break
    err = float(np.abs(back.astype(np.float64) - u).max() / np.abs(u).max())
    t = float(np.mean(times))
    nbytes = u.size * S
    return {"value": 2 * nbytes / t / 1e9, "unit": "GB/s", "cores": cores,
            "kind": "reference" if kind.startswith("reference") else "port",
            "sample": f"{'x'.join(map(str, shape))} {cfg['dtype']} "
                      f"{'nonuniform' if cfg['nonuniform'] else 'uniform'} smooth+noise block"
                      f"{' (the full workload)' if full else ' (bounded sample of the workload)'}, "
                      f"decompose+recompose, mean of {len(times)} x {t:.2f} s "
                      f"({_describe(kind)}, HGR_THREADS={cores})",
            "ms_per_step": t * 1e3, "t_dec_ms": float(np.mean(t_dec)) * 1e3,
            "t_rec_ms": float(np.mean(t_rec)) * 1e3, "roundtrip_rel_err": err, "steps": len(times)}


def run_reference_arm(args, cfg):
    """--impl reference: the reference's CPU implementation on this host's cores,
    on the GPU arm's configuration, K timed round trips (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r = cpu_reference_run(cfg, steps=args.steps, warmup=args.warmup, full=not args.ref_sample)
    line = {"impl": "reference", "metric": "refactor GB/s (decompose+recompose)",
            "value": r["value"], "unit": "GB/s", "n_gpus": args.gpus, "steps": r["steps"],
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic smooth+noise field (SURVEY.md §8d)",
            "config": {"workload": cfg["workload"], "shape": list(cfg["shape"]), "sample": r["sample"],
                       "warmup": f"{args.warmup} round trips of {'x'.join(map(str, cfg['sample']))}"},
            "t_dec_ms": r["t_dec_ms"], "t_rec_ms": r["t_rec_ms"],
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "roundtrip_rel_err": r["roundtrip_rel_err"]}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------

def allreduce(vals, op, device=None):
    """MAX / SUM of a few float64 values over the ranks (no-op for one rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]


def ncu_step(config_name):
    """Whole-step DRAM bytes and kernel time of one round trip from the committed
    ncu launch list (profiles/ncu_traffic.json, tools/make_traffic.py)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(config_name, {}).get("_step")
    except ValueError:
        return None


def measure_device(name, cfg, dev, world, rank, args, red_dev, sample_clocks):
    """Device-resident round trips of one configuration: the measured region
    (graph replays), per-direction times, per-kernel-class times (an identical
    instrumented region), roofline figures. Inputs stay resident in HBM."""
    import torch
    import torch.distributed as dist
    import paper_2007_04457_b200 as hgr

    shape, dt = cfg["shape"], cfg["dtype"]
    coords = coords_for(shape, cfg["nonuniform"])
    g = hgr.GridHierarchy(coords) if coords else hgr.GridHierarchy.uniform(list(shape))
    L = g.levels()
    plan = hgr.Plan(g, dt)
    x = hgr.synthetic_field(shape, dt, seed=shard_seed(rank), device=dev)
    x0 = x.clone()
    P = torch.empty_like(x)
    S = x.element_size()
    nbytes = x.numel() * S
    stream = torch.cuda.current_stream(dev)

    tune_info = None  # tile-segment autotuning, outside every timed region
    if not args.no_autotune:
        t0 = time.perf_counter()
        rep = plan.autotune(x, P)
        torch.cuda.synchronize(dev)
        ents = rep["kernels"]
        tune_info = {"seconds": round(time.perf_counter() - t0, 3), "kernels_tuned": len(ents),
                     "changed": sum(1 for e in ents if e["chosen_s0"] != e["heuristic_s0"])}

    def step():
        plan.decompose_into(x, P)
        plan.recompose_into(P, x, L)

    # one clean round trip (no drift): P = dec(x0), y = rec(P); error on the device
    y = torch.empty_like(x)
    plan.decompose_into(x0, P)
    plan.sync_status()
    plan.recompose_into(P, y, L)
    rt = hgr.error_report(x0, y)
    del y
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed_region():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return ev0.elapsed_time(ev1) / args.steps

    sampler = ClockSampler(dev.index) if sample_clocks else None
    if sampler:
        sampler.start()
    ms_step = timed_region()
    clocks = sampler.stop() if sampler else None

    # per direction (SURVEY §8d timing protocol): events around each decompose
    # and each recompose, median over the steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    for e in evs:
        e[0].record(stream)
        plan.decompose_into(x, P)
        e[1].record(stream)
        plan.recompose_into(P, x, L)
        e[2].record(stream)
    torch.cuda.synchronize(dev)
    t_dec = float(np.median([e[0].elapsed_time(e[1]) for e in evs]))
    t_rec = float(np.median([e[1].elapsed_time(e[2]) for e in evs]))

    # an identical region with per-launch CUDA events on the launching stream
    # (direct launches) gives each kernel class's time for the roofline
    plan.set_profiling(True)
    ms_step_prof = timed_region()
    prof = plan.read_profile()
    plan.set_profiling(False)
    launches_step = plan.launches(0, L) + plan.launches(1, L)

    ms_max, t_dec_max, t_rec_max, err_max = allreduce([ms_step, t_dec, t_rec, rt.linf_rel], "max", red_dev)
    (chk_sum,) = allreduce([float(x.double().sum().item())], "sum", red_dev)
    value = world * 2 * nbytes / (ms_max * 1e-3) / 1e9

    peak, peak_src = measured_peak()
    kinds = {k: v for k, v in prof.items() if v[2] > 0}
    dom = max(kinds, key=lambda k: kinds[k][0])  # dominant kernel class by measured time
    dms, dbytes, dlaunch = kinds[dom]
    achieved = dbytes / (dms * 1e-3) / 1e9
    alg = 2 * algorithmic_bytes(shape, S)
    ncu = ncu_step(name)
    res = {
        "value": round(value, 3), "ms_per_step": round(ms_max, 4),
        "t_dec_ms": round(t_dec_max, 4), "t_rec_ms": round(t_rec_max, 4),
        "refactor_GBps": {"decompose": round(world * nbytes / (t_dec_max * 1e-3) / 1e9, 1),
                          "recompose": round(world * nbytes / (t_rec_max * 1e-3) / 1e9, 1)},
        "config": {"workload": cfg["workload"], "shape": list(shape), "levels": L,
                   "grid": "nonuniform" if cfg["nonuniform"] else "uniform",
                   "bytes_per_gpu": nbytes, "parallelism": f"independent blocks x{world}",
                   "l2": "working set (input %.2f GB) exceeds the 126 MB L2; no flush" % (nbytes / 1e9)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(name, dom), "peak_source": peak_src,
                     "launches_in_timed_region": dlaunch,
                     "algorithmic_bytes_per_launch": dbytes / max(dlaunch, 1)},
        "step_roofline": {"model": "SURVEY.md §8(d) reference-step bytes, both directions "
                                   "(the fused schedule moves fewer, so frac may exceed 1)",
                          "bytes_per_step": alg,
                          "achieved": round(alg / (ms_max * 1e-3) / 1e9, 1),
                          "frac": round(alg / (ms_max * 1e-3) / 1e9 / peak, 4),
                          "compulsory_frac": round(2 * 2 * nbytes / (ms_max * 1e-3) / 1e9 / peak, 4)},
        "dram_frac": None if not ncu else {
            "what": "measured DRAM bytes of one round trip (ncu launch list, profiles/ncu_traffic.json) "
                    "/ ms_per_step / peak: the fraction of HBM bandwidth the step actually moves",
            "dram_bytes_per_step": ncu["dram_bytes"],
            "frac": round(ncu["dram_bytes"] / (ms_max * 1e-3) / 1e9 / peak, 4),
            "source": ncu.get("source")},
        "kernel_timing": {"region": "identical second timed region, per-launch CUDA events, "
                                    "direct launches (the measured region replays CUDA graphs)",
                          "ms_per_step": round(ms_step_prof, 4)},
        "kernels": {k: {"ms_per_step": round(v[0] / args.steps, 4),
                        "GBps": round(v[1] / (v[0] * 1e-3) / 1e9, 1) if v[0] > 0 else None,
                        "launches_per_step": v[2] / args.steps} for k, v in kinds.items()},
        "gpu_launches": launches_step * args.steps,
        "autotune": tune_info,
        "roundtrip_rel_err": err_max,
        "checksum": chk_sum,
    }
    if clocks is not None:
        res["clocks"] = clocks
    del plan, x, x0, P
    torch.cuda.empty_cache()
    return res, g, nbytes


def measure_e2e_host(cfg, g, dev, world, rank, args, red_dev):
    """End to end through the reference-facing host API: hgr_decompose_host_*
    (the reference's decompose(ndarray) consumes its array, so the field buffer
    becomes the pyramid in place) then hgr_recompose_host_* into a second host
    buffer, both pinned; every step moves the field and the pyramid host ->
    device and the pyramid and the reconstruction device -> host. The two
    buffers swap roles each step (the reconstruction is the next step's field).
    The calls are synchronous, so the host clock brackets the whole transfer +
    compute path; max over ranks."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    import paper_2007_04457_b200 as hgr
    from paper_2007_04457_b200 import _lib

    shape, dt = cfg["shape"], cfg["dtype"]
    lib = _lib.load()
    dec = getattr(lib, f"hgr_decompose_host_{dt}")
    rec = getattr(lib, f"hgr_recompose_host_{dt}")
    field = hgr.synthetic_field(shape, dt, seed=shard_seed(rank), device=dev)
    bufs = [torch.empty(tuple(shape), dtype=field.dtype, pin_memory=True) for _ in range(2)]
    bufs[0].copy_(field)
    orig = bufs[0].clone() if args.steps <= 0 else None
    del field
    torch.cuda.empty_cache()
    L = g.levels()
    nbytes = bufs[0].numel() * bufs[0].element_size()

    def one(a, b):
        hgr._check(dec(C.byref(g.desc), a.data_ptr()))
        hgr._check(rec(C.byref(g.desc), a.data_ptr(), b.data_ptr(), L))

    one(bufs[0], bufs[1])  # warm: plan, device buffers, staging
    bufs[0], bufs[1] = bufs[1], bufs[0]
    steps = max(1, min(args.steps, args.e2e_steps))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one(bufs[0], bufs[1])
        bufs[0], bufs[1] = bufs[1], bufs[0]
    t = (time.perf_counter() - t0) / steps
    (t_max,) = allreduce([t], "max", red_dev)
    del bufs, orig
    return {"value": round(world * 2 * nbytes / t_max / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": 2 * nbytes, "d2h_bytes_per_step": 2 * nbytes,
            "ms_per_step": round(t_max * 1e3, 2), "steps": steps,
            "path": "reference-facing host API (C ABI hgr_decompose_host_* + hgr_recompose_host_*, "
                    "what the hgr:: C++ templates call): pinned host field -> device -> pyramid -> "
                    "host, pinned pyramid -> device -> reconstruction -> host, every step; host clock "
                    "around the synchronous calls"}


def measure_e2e_pipelined(cfg, dev, world, rank, args, red_dev):
    """Secondary: device Plan API with the next step's host->device copy on a
    copy stream overlapping the current step's compute; the round-trip error
    scalar comes back each step (the field and pyramid stay on the device)."""
    import torch
    import torch.distributed as dist
    import paper_2007_04457_b200 as hgr

    shape, dt = cfg["shape"], cfg["dtype"]
    coords = coords_for(shape, cfg["nonuniform"])
    g = hgr.GridHierarchy(coords) if coords else hgr.GridHierarchy.uniform(list(shape))
    L = g.levels()
    plan = hgr.Plan(g, dt)
    x0 = hgr.synthetic_field(shape, dt, seed=shard_seed(rank), device=dev)
    stream = torch.cuda.current_stream(dev)
    host = torch.empty(x0.shape, dtype=x0.dtype, pin_memory=True)
    host.copy_(x0)
    xin = [x0, torch.empty_like(x0)]
    P, yout = torch.empty_like(x0), torch.empty_like(x0)
    nbytes = x0.numel() * x0.element_size()
    steps = max(1, min(args.steps, args.e2e_steps))
    copy_stream = torch.cuda.Stream(dev)
    ev_copy = [torch.cuda.Event(), torch.cuda.Event()]
    ev_free = [torch.cuda.Event(), torch.cuda.Event()]
    plan.decompose_into(x0, P)  # warm (graphs)
    plan.recompose_into(P, yout, L)
    plan.decompose_into(x0, P)
    plan.recompose_into(P, yout, L)
    for b in range(2):
        ev_free[b].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def h2d(k):
        b = k % 2
        copy_stream.wait_event(ev_free[b])
        with torch.cuda.stream(copy_stream):
            xin[b].copy_(host, non_blocking=True)
        ev_copy[b].record(copy_stream)

    ea.record(stream)
    copy_stream.wait_event(ea)
    h2d(0)
    for k in range(steps):
        b = k % 2
        if k + 1 < steps:
            h2d(k + 1)
        stream.wait_event(ev_copy[b])
        plan.decompose_into(xin[b], P)
        plan.recompose_into(P, yout, L)
        err_d = (yout - xin[b]).abs().max()
        ev_free[b].record(stream)
        err_d.to("cpu", non_blocking=False)
    eb.record(stream)
    torch.cuda.synchronize(dev)
    (ms,) = allreduce([ea.elapsed_time(eb) / steps], "max", red_dev)
    del plan, host, xin, P, yout
    torch.cuda.empty_cache()
    return {"value": round(world * 2 * nbytes / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": x0.element_size(),
            "ms_per_step": round(ms, 3), "steps": steps,
            "path": "device Plan API, pinned field -> device (next step's copy overlapping this "
                    "step's compute), decompose + recompose, max |error| scalar -> host"}


def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # one process per GPU; HGR_BENCH_BACKEND=gloo lets several ranks share one GPU
    # (a functional check of the multi-rank path on a single-GPU box)
    backend = os.environ.get("HGR_BENCH_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    red_dev = dev if backend == "nccl" else None

    main, g, nbytes = measure_device(args.config, cfg, dev, world, rank, args, red_dev, True)
    e2e = measure_e2e_host(cfg, g, dev, world, rank, args, red_dev)
    e2e_pipe = measure_e2e_pipelined(cfg, dev, world, rank, args, red_dev)
    extra = {}
    # the north-star roofline configuration (1025^3 fp64, BASELINE configs[2]) is
    # measured in the same invocation at N = 1
    if world == 1 and args.config == DEFAULT_CONFIG and not args.no_extra:
        for name in EXTRA_CONFIGS:
            r, _, _ = measure_device(name, CONFIGS[name], dev, world, rank, args, red_dev, False)
            r.pop("checksum", None)
            extra[name] = r

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": "refactor GB/s (decompose+recompose)",
        "value": main.pop("value"), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": main.pop("ms_per_step"), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic smooth+noise field generated on device (SURVEY.md §8d), seed 12345+rank",
        "config": main.pop("config"),
    }
    line.update(main)
    line["e2e"] = e2e
    line["e2e_device_pipelined"] = e2e_pipe
    if extra:
        line["extra_configs"] = extra
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference_run(cfg, seconds_budget=args.cpu_seconds)
        for k in ("ms_per_step", "roundtrip_rel_err", "steps"):
            line["cpu_baseline"].pop(k, None)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch as N ranks (one process
    per GPU) under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=DEFAULT_CONFIG)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="budget of the cpu_baseline sample (rank 0, N=1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-autotune", action="store_true",
                    help="keep the built-in segment heuristics (skip Plan.autotune)")
    ap.add_argument("--ref-sample", action="store_true",
                    help="--impl reference: time the bounded sample instead of the full workload")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the extra 1025^3 fp64 configuration of the default run")
    ap.add_argument("--e2e-steps", type=int, default=5,
                    help="round trips of the end-to-end (host API) measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
