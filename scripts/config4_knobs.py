"""configs[4] (E = 48^3, N = 9, 3 components) batched Helmholtz PCG: time of a
fixed 23-iteration solve (tol 0, CUDA events, best of 3) under CG-vector
knob settings (nk_set_knob 5 = NK_KNOB_CG_PIPE), batched vs sequential.
    python scripts/config4_knobs.py [--pipes 6,2,0]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pipes", default="6,2,0")
ap.add_argument("--ne", type=int, default=48)
ap.add_argument("--N", type=int, default=9)
a = ap.parse_args()
L = _lib.lib()
N, ne = a.N, a.ne
lam0, lam1 = 1.0 / 1000.0, (11.0 / 6.0) / 1e-3
m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
n = m.n_local
b3 = torch.empty((3, n), dtype=torch.float64, device="cuda")
gs = None
for pipe in (int(x) for x in a.pipes.split(",")):
    old = L.nk_set_knob(5, pipe)
    for batched in (True, False):
        hs = nk.HelmholtzVectorSolver(m, lam0, lam1, gs=gs, tol=0.0, max_iter=23, chunk=23,
                                      batched=batched)
        gs = hs.op.gs
        for c in range(3):
            g = torch.Generator(device="cuda").manual_seed(5 + c)
            b3[c] = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
            nk.gs_op(gs, b3[c])
        b3 *= m.mask.reshape(1, -1).to(torch.float64)
        ts = []
        for rep in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hs.solve(b3.reshape((3,) + m.field_shape()))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(json.dumps({"N": N, "E": m.E, "cg_pipe": pipe, "batched": batched,
                          "ms_23_iter": round(min(ts[1:]), 3)}),
              flush=True)
        del hs
        torch.cuda.empty_cache()
    L.nk_set_knob(5, old)
