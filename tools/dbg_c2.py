"""Debug helper: which compact coarse values does a level's Thomas leave unwritten?
Fills the plan workspace with NaN first (via a poisoned earlier plan)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_04457_b200 as hgr
shape = tuple(int(v) for v in sys.argv[1].split('x')); dt = sys.argv[2]
tdt = torch.float64 if dt == 'f64' else torch.float32
# allocate+free a NaN-filled device block of the plan's workspace size so cudaMalloc reuses it
g = hgr.GridHierarchy.uniform(list(shape))
p0 = hgr.Plan(g, dt); ws = p0.workspace_bytes; del p0
import ctypes
lib = ctypes.CDLL('libcudart.so') if False else None
blk = torch.full((ws // (8 if dt == 'f64' else 4) + 1024,), float('nan'), dtype=tdt, device='cuda')
ptr = blk.data_ptr(); del blk; torch.cuda.empty_cache()
p = hgr.Plan(g, dt)
x = hgr.synthetic_field(list(shape), dt, seed=1, device='cuda'); o = torch.empty_like(x)
p.decompose_into(x, o); torch.cuda.synchronize()
print('nonfinite in output:', int((~torch.isfinite(o)).sum()))
