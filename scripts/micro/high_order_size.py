"""BK5 at N = 12..15 vs element count (is the sweep point size-limited?):
pencil (3) and pencil2 (5), cold L2, % of the measured HBM peak."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from bk5_sweep import peak, time_bk5  # noqa: E402
from paper_2104_05829_b200._lib import lib  # noqa: E402

L = lib()
pk = peak()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
for N in (12, 14, 15):
    for ne in (10, 14, 18):
        m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
        for v in (3, 5):
            L.nk_bk5_set_variant(v)
            med, _, _ = time_bk5(nk, L, m, 30, flush)
            frac = 64 * m.n_local / med / 1e6 / pk
            print(json.dumps({"N": N, "E": m.E, "variant": v, "ms": round(med, 4),
                              "frac": round(frac, 3)}), flush=True)
        del m
L.nk_bk5_set_variant(0)
