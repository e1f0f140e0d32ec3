#!/usr/bin/env python
"""Per-part device time of one p-multigrid V-cycle (CUDA events, eager):
fine-level smoothing + residuals, each coarser level, the coarse solve.

    python scripts/prof_vcycle.py [--counts 64 64 64] [--order 7] [--smoother ras]
                                  [--precision 32] [--coarse auto]
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
    ap.add_argument("--counts", nargs=3, type=int, default=[64, 64, 64])
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--smoother", default="ras")
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--coarse", default="auto")
    ap.add_argument("--coarse-tol", type=float, default=1e-3)
    args = ap.parse_args()
    import torch
    import paper_2104_05829_b200 as nk
    m = nk.build_box_mesh((1, 1, 1), tuple(args.counts), args.order, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    t0 = time.perf_counter()
    h = nk.MultigridHierarchy(op, smoother=args.smoother, smoother_precision=args.precision,
                              coarse=args.coarse, coarse_tol=args.coarse_tol)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    r = torch.randn(op.n, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, r)
    r *= m.mask.reshape(-1).to(r.dtype)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    out = {"E": m.E, "N": args.order, "smoother": args.smoother, "precision": args.precision,
           "setup_s": round(setup, 2), "orders": h.orders,
           "coarse": "pcg" if h.levels[-1].cpcg is not None else "dense",
           "coarse_dofs": h.levels[-1].nu}
    out["vcycle_ms"] = round(timed(lambda: h.apply(r)), 3)
    c = h.levels[-1]
    rc = torch.zeros(c.n, dtype=torch.float64, device="cuda")
    rc.normal_()
    nk.gs_op(c.op.gs, rc)
    rc *= c.mask.to(rc.dtype)
    out["coarse_solve_ms"] = round(timed(lambda: h._coarse(c, rc, None)), 3)
    if c.cpcg is not None:
        from paper_2104_05829_b200.solvers import read_state
        h._coarse(c, rc, None)
        out["coarse_pcg_iterations"] = int(read_state(c.cpcg.st).iter)
    for k, lv in enumerate(h.levels):
        out[f"A_level{k}_ms"] = round(timed(lambda lv=lv: lv.op.apply(lv.e, lv.Aq)), 3)
        if lv.sm is not None:
            out[f"smooth_level{k}_ms"] = round(timed(lambda lv=lv: lv.sm.apply(lv.r if lv.r is not None else r, lv.d)), 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
