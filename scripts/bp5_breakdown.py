"""In-situ per-kernel breakdown of one BP5 iteration (FusedPCG.profile_iteration)
at the configs[1] sweep sizes:  python scripts/bp5_breakdown.py [orders]"""
import json, os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "scripts"))
import torch
import paper_2104_05829_b200 as nk
from bk5_sweep import E_FOR_N
orders = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else (5, 7, 8, 11, 14)
for N in orders:
    ne = E_FOR_N[N]
    m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=100, chunk=100)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b); b *= m.mask.reshape(-1).to(torch.float64)
    s.solve(b); s.init(b)
    for _ in range(2): s._iteration()
    print(N, m.n_local, {k: round(x, 4) for k, x in s.profile_iteration().items()})
