"""Decompose / recompose with a NaN-poisoned workspace (HGR_POISON_WORKSPACE=1)."""
import os, sys
os.environ["HGR_POISON_WORKSPACE"] = "1"
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_04457_b200 as hgr
for spec in sys.argv[1:]:
    shp, dt = spec.split(':')
    shape = [int(v) for v in shp.split('x')]
    g = hgr.GridHierarchy.uniform(shape)
    p = hgr.Plan(g, dt)
    x = hgr.synthetic_field(shape, dt, seed=1, device='cuda'); o = torch.empty_like(x); y = torch.empty_like(x)
    p.decompose_into(x, o); p.recompose_into(o, y, g.levels()); torch.cuda.synchronize()
    print(spec, 'nonfinite dec', int((~torch.isfinite(o)).sum()), 'rec', int((~torch.isfinite(y)).sum()),
          'rt', float((y.double() - x.double()).abs().max()))
