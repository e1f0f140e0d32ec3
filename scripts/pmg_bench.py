#!/usr/bin/env python
"""p-multigrid PCG vs Jacobi-PCG time to solution on one GPU (BP5 problem:
deformed box, Dirichlet, N = 7 unless --order), one JSON line per case.

    python scripts/pmg_bench.py [--counts 4 4 4 20 20 20] [--order 7] [--tol 1e-8]
                                [--smoothers cheby_jac asm ras cheby_asm cheby_ras]

Schwarz smoothers run flexible PCG (the counting weight makes them
non-symmetric); each line also carries the in-situ time of one nk_fdm launch
on the fine level (CUDA events, L2 warm) with its flop and byte rates.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rhs(nk, m, gsh):
    import numpy as np
    import torch
    xyz = m.xyz.reshape(3, -1)
    f = 3 * np.pi ** 2 * torch.sin(np.pi * xyz[0]) * torch.sin(np.pi * xyz[1]) * \
        torch.sin(np.pi * xyz[2])
    b = f * m.B.reshape(-1)
    nk.gs_op(gsh, b)
    return b * m.mask.reshape(-1).to(b.dtype)


def timed(solver, b, reps=3):
    import torch
    solver.solve(b)
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        res = solver.solve(b)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        best = t if best is None else min(best, t)
    return res, best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--counts", nargs="*", type=int, default=[4, 4, 4, 20, 20, 20])
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--chunk", type=int, default=4)
    ap.add_argument("--out", default=None)
    ap.add_argument("--smoothers", nargs="*", default=["cheby_jac"])
    ap.add_argument("--precision", type=int, default=64, help="Schwarz local-solve precision")
    ap.add_argument("--coarse", default="auto")
    ap.add_argument("--coarse-tol", nargs="*", type=float, default=[1e-2])
    ap.add_argument("--coarse-iters", type=int, default=50)
    args = ap.parse_args()
    import torch
    import paper_2104_05829_b200 as nk
    N = args.order
    f = open(args.out, "a") if args.out else None
    for q in range(0, len(args.counts), 3):
        counts = tuple(args.counts[q:q + 3])
        m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05), keep_coords=True)
        op = nk.PoissonOperator(m)
        b = rhs(nk, m, op.gs)
        jac = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=args.tol, max_iter=20000,
                          chunk=32)
        rj, tj = timed(jac, b)
        for sm_kind, ctol in [(k, c) for k in args.smoothers for c in args.coarse_tol]:
            flex = sm_kind not in ("jacobi", "cheby_jac")
            t0 = time.perf_counter()
            prec = args.precision if not sm_kind.endswith("jac") and sm_kind != "jacobi" else 64
            h = nk.MultigridHierarchy(op, smoother=sm_kind, smoother_precision=prec,
                                      coarse=args.coarse, coarse_tol=ctol,
                                      coarse_iters=args.coarse_iters)
            torch.cuda.synchronize()
            setup = time.perf_counter() - t0
            s = nk.MultigridPCG(op, h, tol=args.tol, max_iter=2000, chunk=args.chunk,
                                flexible=flex or h.levels[-1].cpcg is not None)
            rm, tm = timed(s, b)
            # per-iteration split: one graph replay of `chunk` iterations
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.init(b)
            a.record()
            s.graph.replay()
            z.record()
            torch.cuda.synchronize()
            ms_it = a.elapsed_time(z) / s.chunk
            dx = float((rm.x - rj.x).abs().max() / rj.x.abs().max())
            line = {"case": "pmg_vs_jacobi", "smoother": sm_kind, "flexible": flex,
                    "smoother_precision": prec,
                    "coarse": "pcg" if h.levels[-1].cpcg is not None else "dense",
                    "coarse_tol": ctol, "coarse_iters": args.coarse_iters,
                    "counts": counts, "E": m.E, "N": N,
                    "dof": m.E * N ** 3, "tol": args.tol,
                    "jacobi_iters": rj.iterations, "jacobi_s": round(tj, 5),
                    "pmg_iters": rm.iterations, "pmg_s": round(tm, 5),
                    "pmg_ms_per_iter": round(ms_it, 4), "pmg_setup_s": round(setup, 3),
                    "coarse_dofs": h.levels[-1].nu, "orders": h.orders,
                    "lmax": [round(lv.lmax, 4) for lv in h.levels[:-1]],
                    "speedup_time_to_solution": round(tj / tm, 3), "max_rel_x_diff": dx,
                    "launches_per_iter": s.launches_per_iter}
            sm0 = h.levels[0].sm
            if sm0 is not None:
                reps = 20
                a.record()
                for _ in range(reps):
                    sm0.fdm(b, sm0.buf, out_ext=sm0.kind == "asm")
                z.record()
                torch.cuda.synchronize()
                t = a.elapsed_time(z) / reps * 1e-3
                nqe = N + 3
                flops = 12 * m.E * nqe ** 4
                sb = 4 if prec == 32 else 8
                byts = m.E * (8 * (N + 1) ** 3 + 12 * 6 * (N + 1) ** 2 + sb * 3 * nqe * (nqe + 1)
                              + 8 * (nqe ** 3 if sm0.kind == "asm" else (N + 1) ** 3))
                line["fdm_us"] = round(t * 1e6, 2)
                line["fdm_gflops"] = round(flops / t * 1e-9, 1)
                line["fdm_gbs"] = round(byts / t * 1e-9, 1)
            print(json.dumps(line), flush=True)
            if f:
                f.write(json.dumps(line) + "\n")
            del s, h
        del jac, op, m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
