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
    for N in [int(x) for x in args.orders.split(",")]:
        for k in [int(x) for x in args.waves.split(",")]:
            m = nk.build_box_mesh((1, 1, 1), (148, k, 1), N, deformation=("sine", 0.05))
            n = m.n_local
            u = torch.randn(n, dtype=torch.float64, device="cuda")
            w = torch.empty_like(u)
            for v in [int(x) for x in args.variants.split(",")]:
                L.nk_bk5_set_variant(v)

                def run():
                    check(L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(u), ptr(w), 1.0, None,
                                   0.0, 1, n, None, None, 0, None, None, 0, 0, sp), "bk5")

                res = {}
                for mode in ("cold", "hot"):
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
                d = {"N": N, "E": m.E, "ctas_per_sm_waves": k, "variant": v,
                     "cold_us": round(1e3 * res["cold"], 2), "hot_us": round(1e3 * res["hot"], 2),
                     "cold_frac": round(bytes_ / res["cold"] / 1e6 / pk, 4),
                     "hot_equiv_frac": round(bytes_ / res["hot"] / 1e6 / pk, 4)}
                print(json.dumps(d), flush=True)
                if out:
                    out.write(json.dumps(d) + "\n")
                    out.flush()
            L.nk_bk5_set_variant(0)
            del m, u, w


if __name__ == "__main__":
    main()
