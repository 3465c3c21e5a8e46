"""Round trips of small shapes that reach every kernel family (for compute-sanitizer)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2007_04457_b200 as hgr
SPECS = sys.argv[1:] or ["8193:f64", "16385:f32", "2049x33:f64", "33x2049:f32", "65x65x65:f32",
                         "33x65x1025:f64", "17x9x5:f64", "129x129:f32"]
for spec in SPECS:
    shp, dt = spec.split(':')
    shape = [int(v) for v in shp.split('x')]
    g = hgr.GridHierarchy.uniform(shape)
    p = hgr.Plan(g, dt)
    x = hgr.synthetic_field(shape, dt, seed=3, device='cuda'); o = torch.empty_like(x); y = torch.empty_like(x)
    p.decompose_into(x, o); p.recompose_into(o, y, g.levels()); p.recompose_into(o, y, max(0, g.levels() - 2))
    q = x.clone(); p.decompose_(q)
    torch.cuda.synchronize()
    print(spec, float((y.double() - x.double()).abs().max()) if g.levels() < 2 else 'ok', flush=True)
