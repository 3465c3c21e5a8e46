import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2007_04457_b200 as hgr, oracle
from tests.synthetic import smooth_field
shape = tuple(int(v) for v in sys.argv[1].split('x')); dt = np.float64 if sys.argv[2] == 'f64' else np.float32
g = hgr.GridHierarchy.uniform(list(shape))
u = smooth_field(shape, dt, 12345)
port = oracle.Oracle("port")
expect = port.decompose(u, None)
x = torch.from_numpy(u).cuda()
plan = hgr.Plan(g, sys.argv[2])
out = torch.empty_like(x)
plan.decompose_into(x, out); plan.sync_status()
e1 = np.abs(out.cpu().numpy() - expect).max()
res = []
for t in range(3):
    ip = x.clone(); plan.decompose_(ip); plan.sync_status()
    a = ip.cpu().numpy()
    res.append((np.isnan(a).sum(), float(np.nanmax(np.abs(a - expect)))))
print(os.environ.get('CFG',''), 'out-of-place err', e1, 'in-place', res)
