"""In-situ DRAM bytes of the BP5 iteration kernels under an L2 knob setting.

Runs eager FusedPCG iterations (E = 20^3, N = 7) so that an ncu pass with
--cache-control none and single-pass metrics sees each kernel with the L2
state the previous kernel left (what the graph-replayed solve sees):
    ncu --cache-control none --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:"tma_pcg|gs_classes|cg_update" -s 30 -c 9 \
        python scripts/prof_bp5_l2.py --l2 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--l2", type=int, default=0)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
L = _lib.lib()
L.nk_set_knob(2, a.l2)
m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
op = nk.PoissonOperator(m)
s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=1000, use_graph=False)
b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
nk.gs_op(op.gs, b)
b *= m.mask.reshape(-1).to(torch.float64)
s.init(b)
for _ in range(a.iters):
    s._iteration()
torch.cuda.synchronize()
print("done", a.l2)
