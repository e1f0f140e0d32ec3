"""A few fused BP5 iterations at order N on the configs[1] sweep size (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import paper_2104_05829_b200 as nk
from bk5_sweep import E_FOR_N  # noqa
N = int(sys.argv[1])
ne = E_FOR_N[N]
m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
op = nk.PoissonOperator(m)
s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=8, chunk=8, use_graph=False)
b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
nk.gs_op(op.gs, b)
b *= m.mask.reshape(-1).to(torch.float64)
s.solve(b)
torch.cuda.synchronize()
