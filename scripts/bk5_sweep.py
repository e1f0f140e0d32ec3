#!/usr/bin/env python
"""BK5 tuning sweep (kernel shapes x L2-prefetch distance, and the N=3..15
sweep of BASELINE configs[1]).  Prints one JSON line per measurement.

    python scripts/bk5_sweep.py [--shapes] [--orders] [--reps 50]

--high-shapes / --seq3-shapes need the sweep build of the library
(cd paper_2104_05829_b200/csrc && make clean && make SWEEP=1).
"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# E per order at ~3M points
E_FOR_N = {1: 96, 2: 64, 3: 48, 4: 36, 5: 29, 6: 24, 7: 20, 8: 18, 9: 16, 10: 14, 11: 13, 12: 12,
           13: 11, 14: 10, 15: 10}


def peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def time_bk5(nk, L, mesh, reps, flush, check_ref=None):
    import numpy as np
    import torch
    from paper_2104_05829_b200._lib import check, ptr
    N, E, n = mesh.N, mesh.E, mesh.n_local
    nq = N + 1
    rng = np.random.default_rng(1000 + N)
    u = torch.as_tensor(rng.standard_normal(n), device="cuda")
    w = torch.empty_like(u)
    D = mesh.basis.diff
    s = torch.cuda.current_stream()
    sp = s.cuda_stream

    def run():
        check(L.nk_bk5(N, E, ptr(D), ptr(mesh.G), ptr(u), ptr(w), 1.0, None, 0.0, 1, n, None,
                       None, 0, None, None, 0, 0, sp), "bk5")

    for _ in range(5):
        L.nk_l2_flush(ptr(flush), flush.numel(), sp)
        run()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        L.nk_l2_flush(ptr(flush), flush.numel(), sp)
        a.record(s)
        run()
        b.record(s)
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ts]
    return statistics.median(ms), min(ms), w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", action="store_true")
    ap.add_argument("--orders", action="store_true")
    ap.add_argument("--low", action="store_true", help="N = 1, 2 variant comparison")
    ap.add_argument("--probe", action="store_true")
    ap.add_argument("--seq3-shapes", default=None,
                    help="comma list of orders: seq3 (3-component) x CTA shapes vs 3 x scalar")
    ap.add_argument("--pf-orders", default=None,
                    help="comma list of orders: auto variant x L2 prefetch mode 0/1/2")
    ap.add_argument("--high-shapes", default=None,
                    help="comma list of orders: pencil / pencil2 x CTA shapes (cfg 0, 11..14)")
    ap.add_argument("--helm3", action="store_true")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_2104_05829_b200 as nk
    from paper_2104_05829_b200 import _lib
    L = _lib.lib()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    pk = peak()
    out = open(args.out, "a") if args.out else None

    def emit(d):
        line = json.dumps(d)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()

    if args.probe:
        m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
        u = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
        w = torch.empty_like(u)
        s = torch.cuda.current_stream()
        from paper_2104_05829_b200._lib import ptr
        for bps in (2, 4, 8, 16, 32):
            ts = []
            for rep in range(args.reps + 5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                L.nk_l2_flush(ptr(flush), flush.numel(), s.cuda_stream)
                a.record(s)
                L.nk_bw_probe(m.E, 512, ptr(u), ptr(m.G), ptr(w), bps, s.cuda_stream)
                b.record(s)
                ts.append((a, b))
            torch.cuda.synchronize()
            ms = statistics.median([a.elapsed_time(b) for a, b in ts[5:]])
            bytes_ = 64 * m.n_local
            emit({"sweep": "probe", "blocks_per_sm": bps, "ms_med": round(ms, 5),
                  "GBs": round(bytes_ / ms / 1e6, 1), "frac": round(bytes_ / ms / 1e6 / pk, 4)})
        # same probe on an 8x larger problem (40^3 elements)
        m2 = nk.build_box_mesh((1, 1, 1), (40, 40, 40), 7, deformation=("sine", 0.05))
        u2 = torch.zeros(m2.n_local, dtype=torch.float64, device="cuda")
        w2 = torch.empty_like(u2)
        for variant in (None, 3, 4):
            ts = []
            for rep in range(args.reps + 5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                if variant is None:
                    L.nk_bw_probe(m2.E, 512, ptr(u2), ptr(m2.G), ptr(w2), 8, s.cuda_stream)
                else:
                    L.nk_bk5_set_variant(variant)
                    L.nk_bk5(7, m2.E, ptr(m2.basis.diff), ptr(m2.G), ptr(u2), ptr(w2), 1.0, None,
                             0.0, 1, m2.n_local, None, None, 0, None, None, 0, 0, s.cuda_stream)
                b.record(s)
                ts.append((a, b))
            torch.cuda.synchronize()
            ms = statistics.median([a.elapsed_time(b) for a, b in ts[5:]])
            bytes_ = 64 * m2.n_local
            emit({"sweep": "probe40", "kernel": "probe" if variant is None else f"bk5 v{variant}",
                  "ms_med": round(ms, 5), "GBs": round(bytes_ / ms / 1e6, 1),
                  "frac": round(bytes_ / ms / 1e6 / pk, 4)})
        L.nk_bk5_set_variant(0)
        del m2, u2, w2
    if args.helm3:
        from paper_2104_05829_b200._lib import ptr
        s = torch.cuda.current_stream()
        for N in range(1, 16):
            ne = E_FOR_N[N]
            m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
            n = m.n_local
            u3 = torch.randn(3 * n, dtype=torch.float64, device="cuda")
            w3 = torch.empty_like(u3)
            lam0, lam1 = 1e-3, 11 / 6 / 1e-3
            def batched():
                L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(u3), ptr(w3), lam0, ptr(m.B),
                         lam1, 3, n, None, None, 0, None, None, 0, 0, s.cuda_stream)
            def separate():
                for c in range(3):
                    L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), u3.data_ptr() + 8 * c * n,
                             w3.data_ptr() + 8 * c * n, lam0, ptr(m.B), lam1, 1, n, None, None,
                             0, None, None, 0, 0, s.cuda_stream)
            def pencil3():
                L.nk_bk5_set_variant(3)
                batched()
                L.nk_bk5_set_variant(0)
            def seq3():
                L.nk_bk5_set_variant(6)
                batched()
                L.nk_bk5_set_variant(0)
            outs = {}
            cands = [("3x scalar", separate, 216), ("seq3", seq3, 104), ("auto", batched, 104)]
            if N <= 11:
                cands.append(("pencil3", pencil3, 104))
            for name, fn, bpp in cands:
                ts = []
                for rep in range(args.reps + 5):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    L.nk_l2_flush(ptr(flush), flush.numel(), s.cuda_stream)
                    a.record(s)
                    fn()
                    b.record(s)
                    ts.append((a, b))
                torch.cuda.synchronize()
                ms = statistics.median([a.elapsed_time(b) for a, b in ts[5:]])
                outs[name] = w3.clone()
                emit({"sweep": "helm3", "N": N, "E": m.E, "kernel": name, "ms_med": round(ms, 5),
                      "bitwise_same_as_scalar": bool(torch.equal(outs["3x scalar"], w3)),
                      "alg_bytes_per_pt": bpp,
                      "frac_of_own_bytes": round(bpp * n / ms / 1e6 / pk, 4),
                      "gdofs_3comp": round(3 * m.E * N ** 3 / ms / 1e6, 3)})
            del m, u3, w3
    if args.shapes:
        m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
        ref = None
        for variant, cfg, pf in [(3, 0, 1), (5, 0, 1), (4, 0, 0)]:
            if True:
                L.nk_bk5_set_variant(variant)
                L.nk_bk5_tune(cfg, pf)
                med, best, w = time_bk5(nk, L, m, args.reps, flush)
                same = None
                if ref is None:
                    ref = w.clone()
                else:
                    same = bool(torch.equal(ref, w))
                bytes_ = 64 * m.n_local
                emit({"sweep": "shape", "variant": variant, "N": 7, "cfg": cfg, "pf": pf, "ms_med": round(med, 5),
                      "ms_best": round(best, 5), "GBs": round(bytes_ / med / 1e6, 1),
                      "frac": round(bytes_ / med / 1e6 / pk, 4),
                      "gdofs": round(m.E * 343 / med / 1e6, 3), "bitwise_same": same})
        L.nk_bk5_tune(0, 0)
        L.nk_bk5_set_variant(0)
    if args.seq3_shapes:
        from paper_2104_05829_b200._lib import ptr
        s = torch.cuda.current_stream()
        for N in [int(x) for x in args.seq3_shapes.split(",")]:
            ne = E_FOR_N[N]
            m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
            n = m.n_local
            u3 = torch.randn(3 * n, dtype=torch.float64, device="cuda")
            w3 = torch.empty_like(u3)
            ref = None
            for kind, cfg in [("3x scalar", 0)] + [("seq3", c) for c in (0, 11, 12, 13, 14)]:
                ts = []
                for rep in range(args.reps + 5):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    L.nk_l2_flush(ptr(flush), flush.numel(), s.cuda_stream)
                    a.record(s)
                    if kind == "seq3":
                        L.nk_bk5_set_variant(6)
                        if L.nk_bk5_tune(cfg, 1) != 0:
                            raise SystemExit(L.nk_last_error().decode())
                        L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(u3), ptr(w3), 1e-3,
                                 ptr(m.B), 1833.3, 3, n, None, None, 0, None, None, 0, 0,
                                 s.cuda_stream)
                        L.nk_bk5_tune(0, 1)
                        L.nk_bk5_set_variant(0)
                    else:
                        for c in range(3):
                            L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), u3.data_ptr() + 8 * c * n,
                                     w3.data_ptr() + 8 * c * n, 1e-3, ptr(m.B), 1833.3, 1, n,
                                     None, None, 0, None, None, 0, 0, s.cuda_stream)
                    b.record(s)
                    ts.append((a, b))
                torch.cuda.synchronize()
                ms = statistics.median([a.elapsed_time(b) for a, b in ts[5:]])
                if ref is None:
                    ref = w3.clone()
                emit({"sweep": "seq3_shape", "N": N, "E": m.E, "kind": kind, "cfg": cfg,
                      "ms_med": round(ms, 5), "close_to_scalar": bool(torch.allclose(ref, w3, rtol=1e-12, atol=1e-9))})
            del m, u3, w3
    if args.pf_orders:
        for N in [int(x) for x in args.pf_orders.split(",")]:
            ne = E_FOR_N[N]
            m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
            for pf in (0, 1, 2):
                L.nk_bk5_tune(0, pf)
                med, best, w = time_bk5(nk, L, m, args.reps, flush)
                emit({"sweep": "pf", "N": N, "E": m.E, "pf": pf, "ms_med": round(med, 5),
                      "frac": round(64 * m.n_local / med / 1e6 / pk, 4)})
            del m
        L.nk_bk5_tune(0, 0)
    if args.high_shapes:
        for N in [int(x) for x in args.high_shapes.split(",")]:
            ne = E_FOR_N[N]
            m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
            ref = None
            combos = [(v, c) for v in (3, 5) for c in (0, 11, 12, 13, 14)]
            if N + 1 in (4, 6, 8):
                combos.append((4, 0))
            for variant, cfg in combos:
                if True:
                    L.nk_bk5_set_variant(variant)
                    if L.nk_bk5_tune(cfg, 1) != 0:
                        raise SystemExit(L.nk_last_error().decode())
                    med, best, w = time_bk5(nk, L, m, args.reps, flush)
                    if ref is None:
                        ref = w.clone()
                    same = bool(torch.equal(ref, w))
                    bytes_ = 64 * m.n_local
                    emit({"sweep": "high_shape", "N": N, "E": m.E, "variant": variant, "cfg": cfg,
                          "ms_med": round(med, 5), "frac": round(bytes_ / med / 1e6 / pk, 4),
                          "gdofs": round(m.E * N ** 3 / med / 1e6, 3), "bitwise_same": same})
            del m
        L.nk_bk5_tune(0, 0)
        L.nk_bk5_set_variant(0)
    if args.orders or args.low:
        low = {1: (0, 1), 2: (0, 3, 5)}
        for N in (range(1, 16) if args.orders else (1, 2)):
            ne = E_FOR_N[N]
            m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
            for variant, pf in (((v, 1) for v in low[N]) if args.low else ((0, 1),)):
                L.nk_bk5_set_variant(variant)
                L.nk_bk5_tune(0, pf)
                med, best, _ = time_bk5(nk, L, m, args.reps, flush)
                bytes_ = 64 * m.n_local
                emit({"sweep": "order", "variant": variant, "pf": pf, "N": N, "E": m.E, "ms_med": round(med, 5),
                      "GBs": round(bytes_ / med / 1e6, 1), "frac": round(bytes_ / med / 1e6 / pk, 4),
                      "gdofs": round(m.E * N ** 3 / med / 1e6, 3),
                      "gflops": round(m.E * (12 * (N + 1) ** 4 + 15 * (N + 1) ** 3) / med / 1e6, 1)})
            del m
        L.nk_bk5_tune(0, 0)
        L.nk_bk5_set_variant(0)


if __name__ == "__main__":
    main()
