#!/usr/bin/env python
"""Projection-based initial guesses over a sequence of slowly varying right-
hand sides (the pressure solve at consecutive time steps):
iterations and time per solve with and without a ProjectionSpace, for
Jacobi-PCG and p-multigrid RAS.  One JSON line per (solver, projection).

    python scripts/projection_bench.py [--counts 20 20 20] [--order 7] [--steps 12]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--counts", nargs=3, type=int, default=[20, 20, 20])
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--capacity", type=int, default=8)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2104_05829_b200 as nk
    m = nk.build_box_mesh((1, 1, 1), tuple(args.counts), args.order, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    mask = m.mask.reshape(-1).to(torch.float64)
    g = torch.Generator(device="cuda").manual_seed(2104)

    def field():
        v = torch.randn(op.n, dtype=torch.float64, device="cuda", generator=g)
        nk.gs_op(op.gs, v)
        return v * op.weights * mask

    # b(t) = b0 + t db1 + t^2 db2 (smooth in "time"), unit-norm pieces
    b0, d1, d2 = field(), field(), field()
    rhs = [b0 + (0.01 * t) * d1 + (0.001 * t * t) * d2 for t in range(args.steps)]
    f = open(args.out, "a") if args.out else None
    for name, make in (("jacobi_pcg", lambda: nk.FusedPCG(op, nk.JacobiPreconditioner(op),
                                                           tol=args.tol, max_iter=5000, chunk=32)),
                       ("pmg_ras", lambda: nk.MultigridPCG(op, nk.MultigridHierarchy(
                           op, smoother="ras", smoother_precision=32), tol=args.tol,
                           max_iter=500))):
        for proj in (False, True):
            sv = make()
            sv.solve(rhs[0])           # warm
            runner = nk.ProjectedSolver(sv, capacity=args.capacity) if proj else sv
            its, ts = [], []
            for b in rhs:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = runner.solve(b)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
                its.append(r.iterations)
                # the answer meets the tolerance against the ORIGINAL rhs
                res = b - op(r.x)
                rel = float(torch.sqrt((op.weights * res * res).sum()) /
                            torch.sqrt((op.weights * b * b).sum()))
                assert rel <= 1.05 * args.tol, rel
            line = {"solver": name, "projection": proj, "capacity": args.capacity if proj else 0,
                    "E": m.E, "N": args.order, "tol": args.tol, "iterations": its,
                    "mean_iterations_after_first": round(float(np.mean(its[1:])), 2),
                    "total_s": round(sum(ts), 4), "ms_per_solve_after_first":
                        round(1e3 * float(np.mean(ts[1:])), 3)}
            print(json.dumps(line), flush=True)
            if f:
                f.write(json.dumps(line) + "\n")
            del sv, runner
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
