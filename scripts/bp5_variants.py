"""BP5 per-iteration time with each fused-step kernel (auto = TMA, 3 = pencil)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2104_05829_b200 as nk
from paper_2104_05829_b200 import _lib
L = _lib.lib()
m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
for v in (0, 3):
    L.nk_bk5_set_variant(v)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    s = nk.FusedPCG(op, jac, tol=1e-30, max_iter=100, chunk=100)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b); b *= m.mask.reshape(-1).to(torch.float64)
    s.solve(b)
    ts = []
    for _ in range(5):
        s.init(b)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); s.graph.replay(); e.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(e) / 100)
    s.init(b)
    for _ in range(2): s._iteration()
    print(json.dumps({"variant": v, "ms_per_iter": round(min(ts), 4),
                      "breakdown": {k: round(x, 4) for k, x in s.profile_iteration().items()}}))
L.nk_bk5_set_variant(0)
# parity across variants: one converged solve each, same iterations / answer
xs = {}
for v in (0, 3):
    L.nk_bk5_set_variant(v)
    op = nk.PoissonOperator(m)
    s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-8, max_iter=2000, chunk=16)
    b = torch.ones(m.n_local, dtype=torch.float64, device="cuda") * m.mask.reshape(-1).to(torch.float64)
    r = s.solve(b)
    xs[v] = (r.iterations, r.x.clone())
L.nk_bk5_set_variant(0)
it0, x0 = xs[0]
print(json.dumps({"iterations": {k: v[0] for k, v in xs.items()},
                  "max_rel_dx": {k: float((v[1] - x0).abs().max() / x0.abs().max()) for k, v in xs.items()}}))
