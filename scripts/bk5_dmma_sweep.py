"""BK5 at high order: FP64 tensor-core kernel (variant 7, bk5_dmma.cuh) vs the
auto table, on the configs[1] sweep sizes (~3M points), cold L2 per launch.
One JSON line per (N, variant): median ms, GB/s at 64 B/pt, fraction of the
measured HBM peak, and the max relative difference of w to the auto kernel.
    python scripts/bk5_dmma_sweep.py [--orders 8,...,15] [--reps 30]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import _lib  # noqa: E402
from bk5_sweep import E_FOR_N, peak, time_bk5  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--orders", default="8,9,10,11,12,13,14,15")
ap.add_argument("--variants", default="0,7")
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
L = _lib.lib()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
pk = peak()
for N in (int(x) for x in a.orders.split(",")):
    ne = E_FOR_N[N]
    m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
    ref = None
    for v in (int(x) for x in a.variants.split(",")):
        old = L.nk_bk5_set_variant(v)
        med, mn, w = time_bk5(nk, L, m, a.reps, flush)
        L.nk_bk5_set_variant(old)
        if ref is None:
            ref = w.clone()
        rel = float((w - ref).abs().max() / ref.abs().max())
        gbs = 64 * m.n_local / med / 1e6
        print(json.dumps({"N": N, "E": m.E, "variant": v, "ms_med": round(med, 5),
                          "ms_min": round(mn, 5), "GBs": round(gbs, 1),
                          "frac": round(gbs / pk, 4), "max_rel_diff_vs_first": rel}), flush=True)
