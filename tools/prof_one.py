"""Autotune, then one warm-up + one measured round trip (for ncu launch lists);
each round trip is preceded by a marker fill kernel. The round trips run inside a
profiler range (cudaProfilerStart/Stop): with `ncu --profile-from-start off` the
tuner's candidate launches are neither profiled nor timed under the profiler,
so the launch list shows the segment lengths bench.py runs with."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2007_04457_b200 as hgr
shape = tuple(int(v) for v in sys.argv[1].split('x')); dt = sys.argv[2]
g = hgr.GridHierarchy.uniform(list(shape))
x = torch.rand(*shape, dtype=torch.float64 if dt == 'f64' else torch.float32, device='cuda')
p_ = torch.empty_like(x)
plan = hgr.Plan(g, dt)
if '--no-tune' not in sys.argv:
    plan.autotune(x, p_)  # as bench.py does
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(2):
    # marker launch (a fill kernel): the tools take the launches after the last one
    torch.ones(1, device='cuda')
    plan.decompose_into(x, p_); plan.recompose_into(p_, x, g.levels())
torch.cuda.synchronize()
torch.cuda.profiler.stop()
