"""Debug helper: decompose of one shape under several tail thresholds vs the oracle."""
import os, subprocess, sys
sys.path.insert(0, '.')
shape = tuple(int(v) for v in sys.argv[1].split('x')); dt = sys.argv[2]
if len(sys.argv) > 3:
    import numpy as np, torch
    import paper_2007_04457_b200 as hgr, oracle
    from tests.synthetic import smooth_field
    # poison: a previous plan's workspace full of NaN (cudaMalloc reuses it)
    gp = hgr.GridHierarchy.uniform([65, 129, 129]); pp = hgr.Plan(gp, dt)
    xp = torch.full((65, 129, 129), float('nan'), dtype=torch.float64 if dt == 'f64' else torch.float32, device='cuda')
    op = torch.empty_like(xp); pp.decompose_into(xp, op); pp.recompose_into(op, xp, gp.levels()); torch.cuda.synchronize()
    del pp
    g = hgr.GridHierarchy.uniform(list(shape))
    u = smooth_field(shape, np.float64 if dt == 'f64' else np.float32, 12345)
    exp = oracle.Oracle('port').decompose(u)
    p = hgr.Plan(g, dt); x = torch.from_numpy(u).cuda(); o = torch.empty_like(x)
    p.decompose_into(x, o); torch.cuda.synchronize()
    got = o.cpu().numpy()
    bad = np.argwhere(~np.isfinite(got))
    err = np.nanmax(np.abs(got.astype(np.float64) - exp))
    print(os.environ.get('HGR_TAIL_NODES'), 'nonfinite', len(bad), bad[:6].tolist(), 'maxerr', err)
else:
    for t in ['0', '1200', '8192']:
        subprocess.run([sys.executable, __file__, sys.argv[1], dt, 'run'], env=dict(os.environ, HGR_TAIL_NODES=t))
