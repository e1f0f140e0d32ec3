#!/usr/bin/env python
"""BK5 cold (L2 flushed) vs hot (L2-resident operands) at the high orders.

For E = k x 148 elements (k CTAs per SM, whole waves), times nk_bk5 with the
L2 flushed between launches and back to back without a flush (u + G + w of
E <= ~2 x 148 elements at N >= 12 stay in the 126 MB L2).  The hot time per
wave is the compute/latency floor of one element per CTA; the cold time per
wave minus it is what the memory stream adds -- the overlap a persistent,
prefetch-ahead kernel could win back.

    python scripts/bk5_hot.py --orders 12,13,14,15 --waves 1,2,4 [--variant V]
"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default="12,13,14,15")
    ap.add_argument("--waves", default="1,2,4")
    ap.add_argument("--variants", default="0")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--cfgs", default="0", help="nk_bk5_tune shape configs (21: stage alt)")
    ap.add_argument("--sweep", action="store_true",
                    help="configs[1] sizes (~3M points, E_FOR_N) instead of whole waves")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_2104_05829_b200 as nk
    from paper_2104_05829_b200._lib import check, lib, ptr
    L = lib()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    sp = s.cuda_stream
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6551.7
    out = open(args.out, "a") if args.out else None
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from bk5_sweep import E_FOR_N
    for N in [int(x) for x in args.orders.split(",")]:
        shapes = ([(E_FOR_N[N],) * 3] if args.sweep else
                  [(148, int(k), 1) for k in args.waves.split(",")])
        for counts in shapes:
            k = counts[1] if not args.sweep else None
            m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
            n = m.n_local
            u = torch.randn(n, dtype=torch.float64, device="cuda")
            w = torch.empty_like(u)
            first = None
            for v, cfg in [(int(x), int(c)) for x in args.variants.split(",")
                           for c in args.cfgs.split(",")]:
                if cfg != 0 and v != 8:
                    continue
                L.nk_bk5_set_variant(v)
                L.nk_bk5_tune(cfg, 1)

                def run():
                    check(L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(u), ptr(w), 1.0, None,
                                   0.0, 1, n, None, None, 0, None, None, 0, 0, sp), "bk5")

                res = {}
                for mode in (("cold",) if args.sweep else ("cold", "hot")):
                    ts = []
                    for rep in range(args.reps + 5):
                        a = torch.cuda.Event(enable_timing=True)
                        b = torch.cuda.Event(enable_timing=True)
                        if mode == "cold":
                            L.nk_l2_flush(ptr(flush), flush.numel(), sp)
                        a.record(s)
                        run()
                        b.record(s)
                        ts.append((a, b))
                    torch.cuda.synchronize()
                    res[mode] = statistics.median([a.elapsed_time(b) for a, b in ts[5:]])
                bytes_ = 64 * n
                if first is None:
                    first = w.clone()
                d = {"N": N, "E": m.E, "ctas_per_sm_waves": k, "variant": v, "cfg": cfg,
                     "cold_us": round(1e3 * res["cold"], 2),
                     "cold_frac": round(bytes_ / res["cold"] / 1e6 / pk, 4),
                     "gdofs": round(m.E * N ** 3 / res["cold"] / 1e6, 2),
                     "bitwise_same_as_first": bool(torch.equal(first, w))}
                if "hot" in res:
                    d["hot_us"] = round(1e3 * res["hot"], 2)
                    d["hot_equiv_frac"] = round(bytes_ / res["hot"] / 1e6 / pk, 4)
                print(json.dumps(d), flush=True)
                if out:
                    out.write(json.dumps(d) + "\n")
                    out.flush()
            L.nk_bk5_set_variant(0)
            L.nk_bk5_tune(0, 1)
            del m, u, w


if __name__ == "__main__":
    main()
