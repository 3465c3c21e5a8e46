"""Print the autotuner's measured candidates for the top fused levels (development aid).
usage: tune_report.py 1025x1025x1025:f32 [repeats]"""
import sys, json
sys.path.insert(0, '.')
import torch
import paper_2007_04457_b200 as hgr

spec = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
shape, dt = spec.split(':')
shape = tuple(int(v) for v in shape.split('x'))
g = hgr.GridHierarchy.uniform(list(shape))
x = torch.rand(*shape, dtype=torch.float64 if dt == 'f64' else torch.float32, device='cuda')
out = torch.empty_like(x)
p = hgr.Plan(g, dt)
for r in range(reps):
    rep = p.autotune(x, out)
    for k in rep['kernels'][:6]:
        print(r, k['level'], k['kernel'], 'heur', k['heuristic_s0'], 'chosen', k['chosen_s0'],
              [(c['s0'], c['blocks'], c['measured_us'] and round(c['measured_us'])) for c in k['candidates']])
