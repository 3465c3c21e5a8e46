"""The multi-GPU path with the product kernels: independent
blocks per rank, no collective on the data path. On a one-GPU box the ranks
share cuda:0 and talk over gloo (HGR_BENCH_BACKEND=gloo); the driver's N-GPU
runs use NCCL with one GPU per rank."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _last_json(out):
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


def test_each_rank_matches_oracle(cuda):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29531", str(ROOT / "tests" / "_rank_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = _last_json(r.stdout)
    print(d)
    assert d["world"] == 2
    assert d["decompose_rel_err"] <= 1e-12 and d["roundtrip_rel_err"] <= 1e-12


def test_bench_spawns_requested_ranks(cuda):
    """`bench.py --gpus 2` outside torchrun launches two ranks itself and
    reports n_gpus = 2 with the aggregate (weak-scaling) value."""
    env = dict(os.environ, HGR_BENCH_BACKEND="gloo")
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", "513f32", "--no-cpu-baseline", "--no-autotune", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["roundtrip_rel_err"] <= 1e-5
    assert "independent blocks x2" in d["config"]["parallelism"]
