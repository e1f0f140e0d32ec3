"""Run BK5 a few times at order N on the configs[1] sweep size (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05829_b200 as nk
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bk5_sweep import E_FOR_N  # noqa
N = int(sys.argv[1])
if len(sys.argv) > 2:   # optional forced variant (nk_bk5_set_variant)
    from paper_2104_05829_b200 import _lib
    _lib.lib().nk_bk5_set_variant(int(sys.argv[2]))
ne = E_FOR_N[N]
m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
u = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
w = torch.empty_like(u)
for _ in range(4):
    nk.apply_stiffness_local(u, m, out=w)
torch.cuda.synchronize()
