"""3-component BK5 with per-component fused dots (nk_bk5_batch, the batched
Helmholtz PCG's operator launch): seq3 (6) and three scalar launches
(forced 3 -> -1), L2 prefetch modes, per order.  (profiles/r2e_helm3_batch*
also holds a measured-and-removed variant 7, "il3": the three components
interleaved over consecutive CTAs of the scalar kernel so G is read from HBM
once and from L2 twice -- slower than seq3 at every order but N = 10, 11.)

    python scripts/helm3_batch_bench.py [--orders 7 9] [--configs4]

Each case: L2 flushed, CUDA events per launch, median of reps; HBM model
bytes = 48 (G) + 8 (B) + 1 (mask) + 3 x 16 (p in, w out) per local point.
--configs4: the E = 48^3, N = 9 box of BASELINE configs[4]."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200._lib import CG_STATE_BYTES, check, lib, ptr  # noqa: E402

E_FOR = {3: 48, 4: 36, 5: 29, 6: 24, 7: 20, 8: 18, 9: 16, 10: 14, 11: 13, 12: 12, 13: 11,
         14: 10, 15: 10}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", type=int, nargs="*", default=[7, 9])
    ap.add_argument("--configs4", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    L = lib()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(
        __file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    f = open(args.out, "a") if args.out else None
    orders = [9] if args.configs4 else args.orders
    for N in orders:
        ne = 48 if args.configs4 else E_FOR[N]
        m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
        n = m.n_local
        p = torch.randn(3 * n, dtype=torch.float64, device="cuda")
        w = torch.empty_like(p)
        st = torch.zeros(3 * CG_STATE_BYTES, dtype=torch.uint8, device="cuda")
        byts = n * (48 + 8 + 1 + 48)
        for forced, name in ((6, "seq3"), (3, "scalar_x3")):
            for pf in (1, 0, 2):
                old = L.nk_bk5_set_variant(forced)
                L.nk_bk5_tune(0, pf)
                try:
                    nb = int(L.nk_bk5_batch_blocks(N, m.E))
                    part = torch.zeros(3 * (nb + 2), dtype=torch.float64, device="cuda")

                    def run():
                        check(L.nk_bk5_batch(N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(p), ptr(w),
                                             0.001, ptr(m.B), 1833.3, 3, n, ptr(m.mask), None, 0,
                                             ptr(st), ptr(part), nb + 2, 0, nb, s), "bk5_batch")
                    ts = []
                    for i in range(args.reps + 3):
                        L.nk_l2_flush(ptr(flush), flush.numel(), s)
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(
                            enable_timing=True)
                        a.record()
                        run()
                        b.record()
                        torch.cuda.synchronize()
                        if i >= 3:
                            ts.append(a.elapsed_time(b))
                    ms = statistics.median(ts)
                    rec = {"N": N, "E": m.E, "variant": name, "pf": pf, "ms": round(ms, 4),
                           "frac_of_peak_model": round(byts / (ms * 1e-3) / 1e9 / peak, 3),
                           "gdofs_3comp": round(3 * m.E * N ** 3 / ms / 1e6, 2)}
                finally:
                    L.nk_bk5_set_variant(old)
                    L.nk_bk5_tune(0, 1)
                print(json.dumps(rec), flush=True)
                if f:
                    f.write(json.dumps(rec) + "\n")
        del m, p, w
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
