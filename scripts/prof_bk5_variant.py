"""Run nk_bk5 a few times at order N, forced variant V and shape cfg C, on
the configs[1] sweep size (for ncu captures)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import _lib  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bk5_sweep import E_FOR_N  # noqa: E402
N, V = int(sys.argv[1]), int(sys.argv[2])
C = int(sys.argv[3]) if len(sys.argv) > 3 else 0
L = _lib.lib()
L.nk_bk5_set_variant(V)
L.nk_bk5_tune(C, 1)
ne = E_FOR_N[N]
m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
u = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
w = torch.empty_like(u)
for _ in range(4):
    nk.apply_stiffness_local(u, m, out=w)
torch.cuda.synchronize()
