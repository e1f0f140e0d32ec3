"""In-situ time of the order-1 fused PCG step (bk5_n1_pcg + gs + cg_update)
and of the plain order-1 apply at E = 64^3, CUDA events over 200 iterations."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402

m1 = nk.build_box_mesh((1, 1, 1), (64, 64, 64), 1, deformation=("sine", 0.05))
op1 = nk.PoissonOperator(m1)
s1 = nk.FusedPCG(op1, nk.JacobiPreconditioner(op1), tol=1e-30, max_iter=100000, use_graph=False)
b1 = torch.randn(op1.n, dtype=torch.float64, device="cuda")
nk.gs_op(op1.gs, b1)
s1.init(b1)
for _ in range(20):
    s1._iteration()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize()
ev[0].record()
for _ in range(200):
    s1._iteration()
ev[1].record()
torch.cuda.synchronize()
it_us = ev[0].elapsed_time(ev[1]) / 200 * 1e3
u = torch.randn(op1.n_local if hasattr(op1, "n_local") else m1.n_local, dtype=torch.float64,
                device="cuda")
w = torch.empty_like(u)
for _ in range(10):
    op1.apply(u, w)
torch.cuda.synchronize()
ev[0].record()
for _ in range(200):
    op1.apply(u, w)
ev[1].record()
torch.cuda.synchronize()
ap_us = ev[0].elapsed_time(ev[1]) / 200 * 1e3
print(json.dumps({"E": m1.E, "pcg_iteration_us": round(it_us, 2), "apply_us": round(ap_us, 2)}))
