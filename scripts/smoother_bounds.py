"""Chebyshev-Schwarz bound fractions on SPEC.md:541's problem (deformed box,
E = 64, N = 7, tol 1e-8, flexible PCG), with the CPU oracle (oracle/pmg.py):
iterations per smoother kind at the defaults and a sweep of the lower bound
fraction for cheby_asm / cheby_ras.  -> profiles/r2_smoother_bounds.jsonl"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import gs as ogs  # noqa: E402
from oracle import pmg as opmg  # noqa: E402
from oracle import solvers as osol  # noqa: E402


def run(kind, bounds=None, degree=2):
    h = opmg.build_hierarchy((1, 1, 1), (4, 4, 4), 7, deformation=("sine", 0.05), smoother=kind,
                             degree=degree, bounds=bounds)
    lv = h["levels"][0]
    m = lv.mesh
    X = m.xyz.reshape(3, -1)
    b = lv.mask * ogs.gs_op(m.ids, m.B.ravel() * 3 * np.pi ** 2 * np.prod(np.sin(np.pi * X), 0))
    r = osol.pcg(opmg.fine_operator(h), lambda v: opmg.vcycle(h, v), b, tol=1e-8, max_iter=200,
                 flexible=True, weights=lv.wt)
    return r.iterations, [float(v.lmax) for v in h["levels"][:-1]]


out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   "r2_smoother_bounds.jsonl")
with open(out, "w") as f:
    for kind in ("jacobi", "cheby_jac", "asm", "ras", "cheby_asm", "cheby_ras"):
        it, lm = run(kind)
        f.write(json.dumps({"case": "defaults", "smoother": kind, "iterations": it,
                            "lmax": lm}) + "\n")
    for kind in ("cheby_asm", "cheby_ras"):
        for lo in (0.1, 0.25, 0.3, 0.4, 0.5, 0.6):
            it, lm = run(kind, (lo, 1.1))
            f.write(json.dumps({"case": "bounds_sweep", "smoother": kind, "bounds": [lo, 1.1],
                                "iterations": it}) + "\n")
        it, _ = run(kind, (0.1, 1.1), degree=3)
        f.write(json.dumps({"case": "degree3_spec_bounds", "smoother": kind, "iterations": it})
                + "\n")
print(open(out).read())
