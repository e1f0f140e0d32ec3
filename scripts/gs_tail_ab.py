"""BP5 per-iteration time with the edge / vertex gs as the tail of the
persistent N = 7 step (nk_bk5_pcg_gs, FusedPCG(gs_tail=True): 2 launches per
iteration) vs the separate gs pass (3 launches), interleaved in one process.
configs[3] per-GPU box (E = 20^3, N = 7 deformed), 100-iteration graph
replays, best / median of --reps per mode, plus a converged solve whose
iterations and x must agree bit for bit.
    python scripts/gs_tail_ab.py [--counts 20,20,20] > profiles/<tag>_gs_tail_ab.jsonl
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--counts", default="20,20,20")
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--mode2", action="store_true",
                help="NK_KNOB_GS_TAIL = 2 (gs at the start of the update kernel) vs 0")
ap.add_argument("--pdl", default="", help="comma list of NK_KNOB_PDL values to sweep")
a = ap.parse_args()
from paper_2104_05829_b200 import _lib  # noqa: E402
L = _lib.lib()
L.nk_set_knob(7, 1)   # NK_KNOB_GS_TAIL: lets FusedPCG(gs_tail=True) fold the tail
counts = tuple(int(c) for c in a.counts.split(","))
N = 7
m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
g = torch.Generator(device="cuda").manual_seed(7)
b = torch.randn(m.n_local, dtype=torch.float64, device="cuda", generator=g)
op = nk.PoissonOperator(m)
nk.gs_op(op.gs, b)
b *= m.mask.reshape(-1).to(torch.float64)
pdls = [int(v) for v in a.pdl.split(",")] if a.pdl else [None]
for pdl in pdls:
  if pdl is not None:
    old = L.nk_set_knob(0, pdl)
  solvers = {}
  for tail in (True, False):
    if a.mode2:
        L.nk_set_knob(7, 2 if tail else 0)
    s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=100, chunk=100,
                    split_step=False, gs_tail=tail and not a.mode2)
    s.solve(b)   # captures the graph under the current knob
    solvers[tail] = s
  ts = {True: [], False: []}
  for _ in range(a.reps):
    for tail, s in solvers.items():
        s.init(b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ts[tail].append(e0.elapsed_time(e1) / 100)
  if pdl is not None:
    print(json.dumps({"pdl_knob": pdl, "ms_tail": statistics.median(ts[True]),
                      "ms_separate": statistics.median(ts[False])}), flush=True)
    L.nk_set_knob(0, old)
res = {}
for tail in (True, False):
    if a.mode2:
        L.nk_set_knob(7, 2 if tail else 0)
    sc = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-8, max_iter=3000, chunk=16,
                     split_step=False, gs_tail=tail and not a.mode2)
    res[tail] = sc.solve(b)
    print(json.dumps({"N": N, "counts": counts, "gs_tail": tail,
                      "launches_per_iter": solvers[tail].launches_per_iter,
                      "ms_per_iter_best": min(ts[tail]),
                      "ms_per_iter_median": statistics.median(ts[tail]),
                      "profile_ms": solvers[tail].profile_iteration(reps=5),
                      "solve_iterations": res[tail].iterations}), flush=True)
print(json.dumps({"bit_identical": bool(torch.equal(res[True].x, res[False].x)) and
                  res[True].iterations == res[False].iterations,
                  "speedup_median": statistics.median(ts[False]) / statistics.median(ts[True])}))
