"""Worker of tests/test_gpu_multirank.py (run under torch.distributed.run, gloo):
each rank refactors its own independent block (seed 12345 + rank)
through the product API on its GPU (ranks share cuda:0 on a one-GPU box) and
checks it against the CPU oracle; the only collective is the final MAX of the
per-rank errors. Rank 0 prints one JSON line."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np
import torch
import torch.distributed as dist

import bench
import oracle
import paper_2007_04457_b200 as hgr
from tests.synthetic import smooth_field


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    shape, dt = (65, 129, 129), np.float64
    u = smooth_field(shape, dt, bench.shard_seed(rank))
    g = hgr.GridHierarchy.uniform(list(shape))
    r = hgr.decompose(torch.from_numpy(u).cuda(), g)
    got = r.data.cpu().numpy()
    want = oracle.Oracle("port").decompose(u)
    scale = float(np.abs(u).max())
    e_dec = float(np.abs(got - want).max()) / scale
    back = hgr.recompose(r, g.levels()).cpu().numpy()
    e_rt = float(np.abs(back - u).max()) / scale
    t = torch.tensor([e_dec, e_rt], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    chk = torch.tensor([float(got.sum())], dtype=torch.float64)
    dist.all_reduce(chk, op=dist.ReduceOp.SUM)
    if rank == 0:
        print(json.dumps({"world": world, "decompose_rel_err": t[0].item(), "roundtrip_rel_err": t[1].item(),
                          "checksum": chk.item()}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
