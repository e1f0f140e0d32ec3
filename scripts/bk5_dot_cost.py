"""nk_bk5 plain vs with the fused p.Ap (CG state + mask) at the configs[1]
sweep sizes: the cost of the per-CTA partials + last-block reduction.
    python scripts/bk5_dot_cost.py [orders]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200._lib import check, lib, ptr  # noqa: E402
from bk5_sweep import E_FOR_N  # noqa: E402

L = lib()
orders = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 3, 4, 5, 6, 7]
s = torch.cuda.current_stream()
for N in orders:
    ne = E_FOR_N[N]
    m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
    n = m.n_local
    u = torch.randn(n, dtype=torch.float64, device="cuda")
    w = torch.empty_like(u)
    nb = int(L.nk_bk5_blocks(N, m.E, 1))
    part = torch.zeros(nb, dtype=torch.float64, device="cuda")
    st = torch.zeros(256, dtype=torch.uint8, device="cuda")
    res = {}
    for name, stp, mk in (("plain", None, None), ("dot+mask", st, m.mask)):
        def run():
            check(L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(u), ptr(w), 1.0, None, 0.0, 1,
                           n, ptr(mk) if mk is not None else None, None, 0,
                           ptr(stp) if stp is not None else None,
                           ptr(part) if stp is not None else None, 0,
                           nb if stp is not None else 0, s.cuda_stream), "bk5")
        for _ in range(3):
            run()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            run()
            b.record(s)
            ts.append((a, b))
        torch.cuda.synchronize()
        res[name] = round(1e3 * statistics.median([a.elapsed_time(b) for a, b in ts]), 2)
    print(json.dumps({"N": N, "E": m.E, "partials": nb, "us": res}), flush=True)
