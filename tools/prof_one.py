"""One warm-up + one measured round trip (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2007_04457_b200 as hgr
shape = tuple(int(v) for v in sys.argv[1].split('x')); dt = sys.argv[2]
g = hgr.GridHierarchy.uniform(list(shape))
x = torch.rand(*shape, dtype=torch.float64 if dt == 'f64' else torch.float32, device='cuda')
p_ = torch.empty_like(x)
plan = hgr.Plan(g, dt)
for _ in range(2):
    plan.decompose_into(x, p_); plan.recompose_into(p_, x, g.levels())
torch.cuda.synchronize()
