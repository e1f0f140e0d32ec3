"""BP5 fused Jacobi-PCG per order at the configs[1] sweep size (~3M points):
ms per iteration from a 100-iteration CUDA-graph replay (tolerance 1e-30 so
every iteration runs), GDOF*iter/s (E N^3 per iteration) and the fraction of
the measured HBM peak for the fused schedule's algorithmic bytes
(143.8 B per local point at one rank: bk5_pcg 105 + gs edge/vertex pass +
cg_update_gs 36).  One JSON line per order.

    python scripts/bp5_orders.py [--orders 1,2,...] [--out file]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default=",".join(str(n) for n in range(1, 16)))
    ap.add_argument("--out", default=None)
    ap.add_argument("--split", default="auto", choices=("auto", "on", "off"),
                    help="FusedPCG split_step: auto (per-order default), on, off")
    args = ap.parse_args()
    import torch
    import paper_2104_05829_b200 as nk
    from bk5_sweep import E_FOR_N, peak
    pk = peak()
    out = open(args.out, "a") if args.out else None
    for N in [int(x) for x in args.orders.split(",")]:
        ne = E_FOR_N[N]
        m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
        op = nk.PoissonOperator(m)
        split = {"auto": None, "on": True, "off": False}[args.split]
        s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=100, chunk=100,
                        split_step=split)
        b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
        nk.gs_op(op.gs, b)
        b *= m.mask.reshape(-1).to(torch.float64)
        s.solve(b)
        ts = []
        for _ in range(5):
            s.init(b)
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s.graph.replay()
            e.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(e) / 100)
        ms = sorted(ts)[len(ts) // 2]
        d = {"sweep": "bp5_order", "N": N, "E": m.E, "split": s.split,
             "ms_per_iteration": round(ms, 5),
             "gdof_iter_per_s": round(m.E * N ** 3 / ms / 1e6, 3),
             "frac_at_143.8_B_per_pt": round(143.8 * m.n_local / ms / 1e6 / pk, 4)}
        line = json.dumps(d)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()
        del s, op, m


if __name__ == "__main__":
    main()
