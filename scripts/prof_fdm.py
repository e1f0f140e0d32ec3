#!/usr/bin/env python
"""nk_fdm in isolation (for ncu): deformed box, Dirichlet, N = 7 unless
--order; `--reps` launches of the ASM (extended output) FDM on the fine level,
then the same number of full Schwarz applications (fdm + gs + post).

    python scripts/prof_fdm.py [--counts 20 20 20] [--order 7] [--kind asm] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--counts", nargs=3, type=int, default=[20, 20, 20])
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--kind", default="asm")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--fdm-knob", type=int, default=None,
                    help="NK_KNOB_FDM: 1 FP64 tensor cores, 0 CUDA-core line kernel")
    args = ap.parse_args()
    import torch
    import paper_2104_05829_b200 as nk
    if args.fdm_knob is not None:
        from paper_2104_05829_b200._lib import lib
        lib().nk_set_knob(3, args.fdm_knob)
    N = args.order
    m = nk.build_box_mesh((1, 1, 1), tuple(args.counts), N, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    sm = nk.SchwarzSmoother(op, args.kind, precision=args.precision)
    r = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, r)
    z = torch.empty_like(r)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(3):        # warm-up (lazy module loading of every kernel)
        sm.fdm(r, sm.buf, out_ext=args.kind == "asm")
        sm.apply(r, z)
    ev[0].record()
    for _ in range(args.reps):
        sm.fdm(r, sm.buf, out_ext=args.kind == "asm")
    ev[1].record()
    for _ in range(args.reps):
        sm.apply(r, z)
    ev[2].record()
    torch.cuda.synchronize()
    t_fdm = ev[0].elapsed_time(ev[1]) / args.reps
    t_app = ev[1].elapsed_time(ev[2]) / args.reps
    nqe = N + 3
    print(json.dumps({"E": m.E, "N": N, "kind": args.kind, "precision": args.precision,
                      "fdm_knob": args.fdm_knob,
                      "fdm_ms": round(t_fdm, 4),
                      "apply_ms": round(t_app, 4),
                      "fdm_gflops": round(12 * m.E * nqe ** 4 / t_fdm * 1e-6, 1)}))


if __name__ == "__main__":
    main()
