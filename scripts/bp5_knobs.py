"""BP5 per-iteration time under the launch / kernel knobs (nk_set_knob).

For each (PDL, CG_UPDATE) setting: FusedPCG on the configs[3] per-GPU box
(E = 20^3, N = 7 deformed; other orders with --orders), 100-iteration graph
replays (best of 7), plus one converged solve whose iteration count and x
must be bit-identical across settings (the knobs change scheduling only).
    python scripts/bp5_knobs.py [--orders 7,5,9] [--settings pdl:pf[:gather[:l2[:tma[:pipe]]]],...]
        > profiles/<tag>_bp5_knobs.jsonl
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--orders", default="7")
ap.add_argument("--counts", default="20,20,20")
ap.add_argument("--settings", default="0:0,1:0,0:1,1:1")
a = ap.parse_args()
L = _lib.lib()
print(json.dumps({"l2_set_aside_max_bytes": int(L.nk_l2_set_aside_max())}), flush=True)
counts = tuple(int(c) for c in a.counts.split(","))
settings = [tuple(int(v) for v in s.split(":")) for s in a.settings.split(",")]
# pdl:cg_update_pf[:gather[:l2[:tma[:pipe]]]]
settings = [st + (0, 0, 2, 0)[len(st) - 2:] if len(st) < 6 else st for st in settings]

for N in (int(o) for o in a.orders.split(",")):
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    g = torch.Generator(device="cuda").manual_seed(7)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda", generator=g)
    op0 = nk.PoissonOperator(m)
    nk.gs_op(op0.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    ref = None
    for pdl, cgu, gat, l2, tma, pipe in settings:
        old = (L.nk_set_knob(0, pdl), L.nk_set_knob(1, cgu), L.nk_set_knob(2, l2))
        old_tma = L.nk_set_knob(4, tma)
        old_pipe = L.nk_set_knob(5, pipe)
        op = nk.PoissonOperator(m)
        s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=100, chunk=100,
                        gather_segments=bool(gat))
        s.solve(b)
        ts = []
        for _ in range(7):
            s.init(b)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.graph.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 100)
        sc = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-8, max_iter=3000, chunk=16,
                         gather_segments=bool(gat))
        res = sc.solve(b)
        x = res.x.clone()
        if ref is None:
            ref = (res.iterations, x)
        same = res.iterations == ref[0] and bool(torch.equal(x, ref[1]))
        print(json.dumps({"N": N, "E": m.E, "pdl": pdl, "cg_update_pf": cgu,
                          "gather_segments": bool(gat), "l2": l2, "tma": tma, "cg_pipe": pipe, "launches_per_iter": s.launches_per_iter,
                          "split": bool(s.split), "ms_per_iter": round(min(ts), 5),
                          "ms_per_iter_median": round(sorted(ts)[len(ts) // 2], 5),
                          "solve_iterations": res.iterations,
                          "bit_identical_to_first_setting": same}), flush=True)
        for kk, v in enumerate(old):
            L.nk_set_knob(kk, v)
        L.nk_set_knob(4, old_tma)
        L.nk_set_knob(5, old_pipe)
