"""Time in-place vs out-of-place decompose / recompose through the plan API (dev aid)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2007_04457_b200 as hgr
shape = tuple(int(v) for v in sys.argv[1].split('x')); dt = sys.argv[2]
g = hgr.GridHierarchy.uniform(list(shape))
x = torch.rand(*shape, dtype=torch.float64 if dt == 'f64' else torch.float32, device='cuda')
p = torch.empty_like(x); y = torch.empty_like(x)
plan = hgr.Plan(g, dt)
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
print('decompose_into %.3f ms' % t(lambda: plan.decompose_into(x, p)))
z = x.clone()
print('decompose_ (in place) %.3f ms' % t(lambda: plan.decompose_(z)))
print('recompose_into %.3f ms' % t(lambda: plan.recompose_into(p, y, g.levels())))
q = p.clone()
print('recompose in place %.3f ms' % t(lambda: plan.recompose_into(q, q, g.levels())))
