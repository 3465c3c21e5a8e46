"""Dev aid: localise decompose/recompose errors vs the C oracle by level and parity class."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle
import paper_2007_04457_b200 as hgr

shape = tuple(int(v) for v in sys.argv[1].split('x'))
dt = np.float64 if (len(sys.argv) < 3 or sys.argv[2] == 'f64') else np.float32
rng = np.random.default_rng(3)
u = rng.uniform(-1, 1, shape).astype(dt)
port = oracle.Oracle('port')
ref = port.decompose(u)
g = hgr.GridHierarchy.uniform(list(shape))
L = g.levels()
r = hgr.decompose(torch.from_numpy(u).cuda(), g)
got = r.data.cpu().numpy().astype(np.float64)
err = np.abs(got - ref)
print('decompose max err', err.max(), 'L', L)
D = len(shape)
for lvl in range(L, 0, -1):
    s = 1 << (L - lvl)
    sl = tuple(slice(None, None, s) for _ in range(D))
    e = err[sl]
    for par in np.ndindex(*([2] * D)):
        sub = e[tuple(slice(p, None, 2) for p in par)]
        if par == (0,) * D:
            continue
        m = sub.max()
        if m > 1e-9:
            idx = np.unravel_index(np.argmax(sub), sub.shape)
            print(f'  level {lvl} parity {par}: max {m:.3e} at {idx} of {sub.shape}; n>1e-9: {(sub > 1e-9).sum()}')
c0 = err[tuple(slice(None, None, 1 << L) for _ in range(D))]
print('  class 0 max', c0.max())
back = hgr.recompose(hgr.RefactoredArray(torch.from_numpy(ref.astype(dt)).cuda(), g), L)
rb = back.cpu().numpy().astype(np.float64)
print('recompose(oracle pyramid) max err vs u', np.abs(rb - u).max())
