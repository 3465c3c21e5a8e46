"""Ad-hoc timing of decompose/recompose via the plan API (development aid)."""
import sys, json
sys.path.insert(0, '.')
import torch
import paper_2007_04457_b200 as hgr

def run(shape, dt, iters=5):
    g = hgr.GridHierarchy.uniform(list(shape))
    tdt = torch.float64 if dt == 'f64' else torch.float32
    x = torch.rand(*shape, dtype=tdt, device='cuda')
    p_ = torch.empty_like(x)
    p = hgr.Plan(g, dt)
    L = g.levels()
    for _ in range(2):
        p.decompose_into(x, p_); p.recompose_into(p_, x, L)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    td = tr = 0
    for _ in range(iters):
        e[0].record(); p.decompose_into(x, p_); e[1].record(); p.recompose_into(p_, x, L); e[2].record()
        torch.cuda.synchronize(); td += e[0].elapsed_time(e[1]); tr += e[1].elapsed_time(e[2])
    td /= iters; tr /= iters
    nbytes = x.numel() * x.element_size()
    print(json.dumps(dict(shape=shape, dt=dt, dec_ms=round(td, 3), rec_ms=round(tr, 3),
          GBps_roundtrip=round(2 * nbytes / ((td + tr) * 1e-3) / 1e9, 1), ws_GB=p.workspace_bytes / 1e9,
          launches=[p.launches(0, L), p.launches(1, L)])))

for spec in sys.argv[1:]:
    shape, dt = spec.split(':')
    run(tuple(int(v) for v in shape.split('x')), dt)
