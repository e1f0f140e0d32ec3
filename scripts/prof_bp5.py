"""Run a few fused PCG iterations eagerly (for ncu captures of the BP5 kernels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2104_05829_b200 as nk

N = 7
m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), N, deformation=("sine", 0.05))
op = nk.PoissonOperator(m)
jac = nk.JacobiPreconditioner(op)
s = nk.FusedPCG(op, jac, tol=1e-30, max_iter=50, use_graph=False)
rng = np.random.default_rng(1)
b = torch.as_tensor(rng.standard_normal(m.n_local), device="cuda")
nk.gs_op(op.gs, b)
b *= m.mask.reshape(-1).to(torch.float64)
s.init(b)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    s._iteration()
torch.cuda.synchronize()
print("iter", nk.solvers.read_state(s.st).iter)
