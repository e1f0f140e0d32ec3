"""BP5 iteration at E = 20^3, N = 7: fused-gs update (2 kernels) vs the
3-kernel schedule; in-situ breakdown per kernel (eager, CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402

m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
op = nk.PoissonOperator(m)
jac = nk.JacobiPreconditioner(op)
b = torch.randn(op.n, dtype=torch.float64, device="cuda")
nk.gs_op(op.gs, b)
b *= m.mask.reshape(-1).to(b.dtype)
for fuse in (True, False):
    s = nk.FusedPCG(op, jac, tol=1e-30, max_iter=10 ** 6, fuse_gs=fuse, use_graph=False)
    s.init(b)
    for _ in range(5):
        s._iteration()
    prof = s.profile_iteration(reps=20)
    print(json.dumps({"fuse_gs": fuse, "ms": {k: round(v, 4) for k, v in prof.items()}}))
