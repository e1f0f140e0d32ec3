#!/usr/bin/env python
"""One launch of every libnekb200 kernel family at a bandwidth-relevant size
(E = 20^3, N = 7 unless noted), for an ncu metrics pass:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --csv --log-file zoo.csv python scripts/kernel_zoo.py
    python scripts/kernel_zoo.py --summarize zoo.csv   -> profiles/<tag>_kernel_zoo.json

Each launch is bracketed by an L2 flush so the DRAM bytes are the kernel's
own; the summary reports achieved DRAM GB/s and the fraction of the
measured HBM peak (MEASURED_PEAKS.json) per kernel."""
import argparse
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run():
    import numpy as np
    import torch
    import paper_2104_05829_b200 as nk
    from paper_2104_05829_b200._lib import check, lib, ptr, stream_ptr
    L = lib()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")

    def fl():
        flush.fill_(1.0)

    N, c = 7, (20, 20, 20)
    m = nk.build_box_mesh((1, 1, 1), c, N, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m, lam1=0.0)
    n = m.n_local
    u = torch.randn(n, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, u)
    u *= m.mask.reshape(-1).to(u.dtype)
    w = torch.empty_like(u)
    # BK5 variants
    for v in (1, 3, 4, 5):
        L.nk_bk5_set_variant(v)
        fl(); nk.apply_stiffness_local(u, m, out=w)
    L.nk_bk5_set_variant(0)
    # 3-component Helmholtz (pencil3)
    u3 = torch.randn(3 * n, dtype=torch.float64, device="cuda")
    fl(); nk.apply_helmholtz_local(u3, m, 1e-3, 1833.0, ncomp=3)
    # gs (classes), local diag, geometry
    fl(); nk.gs_op(op.gs, w)
    fl(); nk.extract_diagonal(m, assemble=False)
    fl(); nk.build_box_mesh((1, 1, 1), c, N, deformation=("sine", 0.05))
    # fused PCG step + cg kernels
    s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-30, max_iter=10, use_graph=False)
    s.init(u)
    for _ in range(2):
        fl(); s._iteration()
    # p-multigrid (transfers, Chebyshev steps, dense coarse, FDM, Schwarz post)
    for sm, prec in (("cheby_jac", 64), ("ras", 32), ("asm", 64)):
        h = nk.MultigridHierarchy(op, smoother=sm, smoother_precision=prec)
        fl(); h.apply(u)
    # order-1 fused step (coarse solve kernel)
    m1 = nk.build_box_mesh((1, 1, 1), (64, 64, 64), 1, deformation=("sine", 0.05))
    op1 = nk.PoissonOperator(m1)
    s1 = nk.FusedPCG(op1, nk.JacobiPreconditioner(op1), tol=1e-30, max_iter=10, use_graph=False)
    b1 = torch.randn(op1.n, dtype=torch.float64, device="cuda")
    nk.gs_op(op1.gs, b1)
    s1.init(b1)
    for _ in range(2):
        fl(); s1._iteration()
    # projection
    sp = nk.ProjectionSpace(op, capacity=8)
    for q in range(8):
        sp.update(u * (1.0 + 0.1 * q) + 0.01 * q * w)
    fl(); sp.project(u)
    torch.cuda.synchronize()
    print("zoo ok")


def summarize(path, tag):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    launches = {}
    for d in data:
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").strip()
        if not name.startswith("nk::"):            # setup / torch kernels
            continue
        key = (d["ID"], name)
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
                 "nsecond": 1e-9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                 "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        launches.setdefault(key, {})[d["Metric Name"]] = v * scale
    best = {}
    for (lid, k), mv in launches.items():
        t = mv.get("gpu__time_duration.sum")
        by = mv.get("dram__bytes_read.sum", 0) + mv.get("dram__bytes_write.sum", 0)
        if not t:
            continue
        gbs = by / t / 1e9
        cur = best.get(k)
        if cur is None or by > cur["dram_bytes"]:       # the largest launch of the family
            best[k] = {"time_us": round(t * 1e6, 2), "dram_bytes": int(by),
                       "dram_GBs": round(gbs, 1), "frac_of_measured_peak": round(gbs / peak, 3)}
    out = os.path.join(ROOT, "profiles", f"{tag}_kernel_zoo.json")
    json.dump({"peak_GBs": peak, "source": os.path.basename(path), "kernels": best},
              open(out, "w"), indent=1)
    print("wrote", out)
    for k, v in sorted(best.items(), key=lambda x: -x[1]["dram_bytes"]):
        print(f"{k[:60]:60s} {v['time_us']:9.2f} us {v['dram_bytes'] / 1e6:9.1f} MB "
              f"{v['dram_GBs']:8.1f} GB/s {100 * v['frac_of_measured_peak']:5.1f}%")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--summarize", default=None)
    ap.add_argument("--tag", default="r1h")
    a = ap.parse_args()
    if a.summarize:
        summarize(a.summarize, a.tag)
    else:
        run()
