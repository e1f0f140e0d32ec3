"""BP5 per-iteration time, fused one-kernel step vs split step (xpstep +
BK5 with the fused dot), over mesh sizes: where the 4th launch stops paying
(FusedPCG's split_step auto rule).
    python scripts/split_crossover.py [orders] [box edges | 0 = the configs[1] size]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402


def per_iter(op, b, split, iters=100):
    s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=iters, chunk=iters,
                    use_graph=True, split_step=split)
    s.solve(b)
    s.init(b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        s.init(b)
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.graph.replay()
        c.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(c) / iters)
    return best


orders = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [3, 5, 9, 12]
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 6, 8, 12, 16]
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from bk5_sweep import E_FOR_N  # noqa: E402
for N in orders:
    for ne in (sizes if sizes != [0] else [E_FOR_N[N]]):
        m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
        op = nk.PoissonOperator(m)
        b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
        nk.gs_op(op.gs, b)
        b *= m.mask.reshape(-1).to(torch.float64)
        f, sp = per_iter(op, b, False), per_iter(op, b, True)
        print(json.dumps({"N": N, "E": m.E, "n_local": m.n_local, "fused_ms": round(f, 5),
                          "split_ms": round(sp, 5), "split_speedup": round(f / sp, 3)}), flush=True)
