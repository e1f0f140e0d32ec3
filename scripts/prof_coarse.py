"""In-situ per-kernel times of one fused Jacobi-PCG iteration on the order-1
p-multigrid level of a box (the iterative coarse solve)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05829_b200 as nk
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m = nk.build_box_mesh((1, 1, 1), (n, n, n), 1, deformation=("sine", 0.05))
op = nk.PoissonOperator(m)
s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=50, use_graph=False)
b = torch.randn(op.n, dtype=torch.float64, device="cuda")
nk.gs_op(op.gs, b)
b *= m.mask.reshape(-1).to(b.dtype)
s.init(b)
for _ in range(3):
    s._iteration()
out = {k: round(v * 1e3, 2) for k, v in s.profile_iteration().items()}
out.update({"E": m.E, "local_points": m.n_local, "gs_shared": int(op.gs.nperm),
            "gs_segments": int(op.gs.nseg)})
print(json.dumps(out))
