"""Eager BP5 iterations at N = 7, E = 20^3 with and without the gs tail
(NK_KNOB_GS_TAIL), for an ncu launch list of the step / gs / update kernels:
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        python scripts/micro/gs_tail_ncu.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import _lib  # noqa: E402

L = _lib.lib()
m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
op = nk.PoissonOperator(m)
nk.gs_op(op.gs, b)
b *= m.mask.reshape(-1).to(torch.float64)
for knob in (1, 0):
    L.nk_set_knob(7, knob)
    s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=100, use_graph=False,
                    split_step=False)
    s.init(b)
    for _ in range(6):
        s._iteration()
    torch.cuda.synchronize()
    print("knob", knob, "gs_tail", s.gs_tail, flush=True)
