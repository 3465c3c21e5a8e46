"""Dev aid: one decompose + recompose of a given shape (for compute-sanitizer)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2007_04457_b200 as hgr
shape = tuple(int(v) for v in sys.argv[1].split('x')); dt = sys.argv[2]
g = hgr.GridHierarchy.uniform(list(shape))
x = torch.rand(*shape, dtype=torch.float64 if dt == 'f64' else torch.float32, device='cuda')
p = torch.empty_like(x)
plan = hgr.Plan(g, dt)
plan.decompose_into(x, p); torch.cuda.synchronize()
print('decompose ok')
y = torch.empty_like(x)
plan.recompose_into(p, y, g.levels()); torch.cuda.synchronize()
print('recompose ok, max err', (y - x).abs().max().item())
