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
                        sample=(257, 257, 257)),
    "513f32": dict(shape=(513, 513, 513), dtype="f32", nonuniform=False,
                   workload="3D 513^3 fp32 uniform grid, all levels (BASELINE configs[1])",
                   sample=(257, 257, 257)),
    "1025f64": dict(shape=(1025, 1025, 1025), dtype="f64", nonuniform=False,
                    workload="3D 1025^3 fp64 uniform grid roofline run (BASELINE configs[2])",
                    sample=(257, 257, 257)),
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

def cpu_reference_run(cfg, seconds_budget=None, steps=None, warmup=0):
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    os.environ["HGR_THREADS"] = str(cores)
    import oracle
    kind = "reference" if oracle.available("reference") else "port"
    O = oracle.Oracle(kind)
    shape = cfg["sample"]
    coords = coords_for(shape, cfg["nonuniform"])
    u = host_field(shape, cfg["dtype"], 12345)
    S = u.dtype.itemsize
    L = O.levels(shape, coords)
    times = []
    for i in range(warmup):
        O.recompose(O.decompose(u, coords), L, coords)
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        back = O.recompose(O.decompose(u, coords), L, coords)
        times.append(time.perf_counter() - t0)
        if steps is not None and len(times) >= steps:
            break
        if seconds_budget is not None and time.perf_counter() - t_start >= seconds_budget:
            break
    err = float(np.abs(back.astype(np.float64) - u).max() / np.abs(u).max())
    t = float(np.mean(times))
    nbytes = u.size * S
    return {"value": 2 * nbytes / t / 1e9, "unit": "GB/s", "cores": cores, "kind": kind,
            "sample": f"{'x'.join(map(str, shape))} {cfg['dtype']} "
                      f"{'nonuniform' if cfg['nonuniform'] else 'uniform'} smooth+noise block, "
                      f"decompose+recompose, mean of {len(times)} x {t:.2f} s "
                      f"({'oracle/_ref: the unmodified reference headers' if kind == 'reference' else 'oracle port'},"
                      f" HGR_THREADS={cores})",
            "ms_per_step": t * 1e3, "roundtrip_rel_err": err, "steps": len(times)}


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r = cpu_reference_run(cfg, steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": "refactor GB/s (decompose+recompose)",
            "value": r["value"], "unit": "GB/s", "n_gpus": args.gpus, "steps": r["steps"],
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic smooth+noise field (SURVEY.md §8d)",
            "config": {"workload": cfg["workload"], "sample": r["sample"]},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "roundtrip_rel_err": r["roundtrip_rel_err"]}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------

def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_2007_04457_b200 as hgr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; HGR_BENCH_BACKEND=gloo lets several ranks share one GPU
    # (a functional check of the multi-rank path on a single-GPU box)
    backend = os.environ.get("HGR_BENCH_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    red_dev = dev if backend == "nccl" else None

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

    # tile-segment autotuning, outside every timed region
    tune_info = None
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

    # correctness of one clean round trip (no drift): P = dec(x0), y = rec(P)
    y = torch.empty_like(x)
    plan.decompose_into(x0, P)
    plan.sync_status()
    plan.recompose_into(P, y, L)
    rt_err = float(((y.double() - x0.double()).abs().max() / x0.double().abs().max()).item())
    del y
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local)
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

    # the measured region: the plan replays each direction as one CUDA graph
    sampler.start()
    ms_step = timed_region()
    clocks = sampler.stop()
    # an identical second region with per-launch CUDA events on the launching
    # stream (direct launches) gives each kernel class's time for the roofline
    plan.set_profiling(True)
    ms_step_prof = timed_region()
    prof = plan.read_profile()
    plan.set_profiling(False)
    launches_step = plan.launches(0, L) + plan.launches(1, L)

    ms_max, chk_sum = reduce_across_ranks(ms_step, float(x.double().sum().item()), red_dev)
    value = world * 2 * nbytes / (ms_max * 1e-3) / 1e9

    # ---- end to end through the public API: pinned host field -> device, full
    # decompose + recompose, round-trip error metric read back to the host every
    # step. Streaming form: step k+1's host->device copy runs on a copy stream
    # while step k computes (two device input buffers); each step still moves its
    # whole input over PCIe and waits for its own result on the host.
    host = torch.empty(x0.shape, dtype=x0.dtype, pin_memory=True)
    host.copy_(x0)
    xin = [torch.empty_like(x0), torch.empty_like(x0)]
    yout = torch.empty_like(x0)
    e2e_steps = max(1, min(args.steps, 5))
    copy_stream = torch.cuda.Stream(dev)
    ev_copy = [torch.cuda.Event(), torch.cuda.Event()]
    ev_free = [torch.cuda.Event(), torch.cuda.Event()]
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
    for k in range(e2e_steps):
        b = k % 2
        if k + 1 < e2e_steps:
            h2d(k + 1)
        stream.wait_event(ev_copy[b])
        plan.decompose_into(xin[b], P)
        plan.recompose_into(P, yout, L)
        err_d = (yout - xin[b]).abs().max()
        ev_free[b].record(stream)
        err_h = err_d.to("cpu", non_blocking=False)
    eb.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms, _ = reduce_across_ranks(ea.elapsed_time(eb) / e2e_steps, 0.0, red_dev)
    e2e_value = world * 2 * nbytes / (e2e_ms * 1e-3) / 1e9
    del host, xin, yout

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peak()
    # dominant kernel class by measured time
    kinds = {k: v for k, v in prof.items() if v[2] > 0}
    dom = max(kinds, key=lambda k: kinds[k][0])
    dms, dbytes, dlaunch = kinds[dom]
    achieved = dbytes / (dms * 1e-3) / 1e9
    traffic = ncu_traffic(args.config, dom)
    alg = 2 * algorithmic_bytes(shape, S)
    line = {
        "metric": "refactor GB/s (decompose+recompose)",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dt,
        "data": "synthetic smooth+noise field generated on device (SURVEY.md §8d), seed 12345+rank",
        "config": {"workload": cfg["workload"], "shape": list(shape), "levels": L,
                   "grid": "nonuniform" if cfg["nonuniform"] else "uniform",
                   "bytes_per_gpu": nbytes, "parallelism": f"independent blocks x{world}",
                   "l2": "working set (input %.2f GB) exceeds the 126 MB L2; no flush" % (nbytes / 1e9)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "peak_source": peak_src,
                     "launches_in_timed_region": dlaunch,
                     "algorithmic_bytes_per_launch": dbytes / max(dlaunch, 1)},
        "step_roofline": {"model": "SURVEY.md §8(d) reference-step bytes, both directions",
                          "bytes_per_step": alg,
                          "achieved": round(alg / (ms_max * 1e-3) / 1e9, 1),
                          "frac": round(alg / (ms_max * 1e-3) / 1e9 / peak, 4),
                          "compulsory_frac": round(2 * 2 * nbytes / (ms_max * 1e-3) / 1e9 / peak, 4)},
        "kernel_timing": {"region": "identical second timed region, per-launch CUDA events, "
                                    "direct launches (the measured region replays CUDA graphs)",
                          "ms_per_step": round(ms_step_prof, 4)},
        "kernels": {k: {"ms_per_step": round(v[0] / args.steps, 4),
                        "GBps": round(v[1] / (v[0] * 1e-3) / 1e9, 1) if v[0] > 0 else None,
                        "launches_per_step": v[2] / args.steps} for k, v in kinds.items()},
        "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": nbytes,
                "d2h_bytes_per_step": S, "ms_per_step": round(e2e_ms, 3),
                "path": "pinned host field -> device (the next step's copy on a copy "
                        "stream overlapping this step's compute), hgr Plan decompose+recompose, "
                        "max |error| scalar -> host every step", "steps": e2e_steps},
        "gpu_launches": launches_step * args.steps,
        "autotune": tune_info,
        "clocks": clocks,
        "roundtrip_rel_err": rt_err,
        "checksum": chk_sum,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference_run(cfg, seconds_budget=args.cpu_seconds)
        for k in ("ms_per_step", "roundtrip_rel_err", "steps"):
            line["cpu_baseline"].pop(k, None)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
