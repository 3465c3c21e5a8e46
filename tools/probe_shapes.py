import sys, torch, numpy as np
sys.path.insert(0,'.')
import paper_2007_04457_b200 as hgr
for shape in [(129,257,257),(257,257,129),(129,129,257),(65,257,257),(129,513,513),(33,257,513)]:
  for dt in (torch.float32, torch.float64):
    g = hgr.GridHierarchy.uniform(list(shape))
    x = torch.randn(shape, dtype=dt, device='cuda')
    try:
        r = hgr.decompose(x, g); b = hgr.recompose(r, g.levels()); torch.cuda.synchronize()
        print(shape, dt, "ok", float((b-x).abs().max()))
    except Exception as e:
        print(shape, dt, "FAIL", e)
