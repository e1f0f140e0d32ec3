"""Per-config golden fixtures from the CPU oracle (fixed seeds).

    python tests/golden/make_config_golden.py

Each BASELINE.json config gets a small, seeded instance whose oracle outputs
are frozen here, so drift in the oracle (mesh / ids / gs / BK5 / PCG / RCB)
is caught by tests/test_golden_configs.py on CPU and the product is compared
against the same numbers on the GPU (tests/test_gpu_golden.py):

config0_bp5.npz    configs[0] verbatim: BP5 4x4x4, N = 7, deformed and affine,
                   Jacobi PCG tol 1e-8 (ids, mask, rhs, x, iterations, history)
config1_bk5.npz    configs[1] sweep points N = 3, 7, 11, 15 on small deformed
                   boxes: u ~ N(0,1) with default_rng(1000 + N) (as the sweep)
                   and w = A_L u; plus the same at N = 7 with the mass term
config23_part.npz  configs[2]/[3] partitions: RCB of the 64^3 box over 8 ranks
                   and of the 40x20x20 weak-scaling box over 2 ranks, and the
                   multi-rank gs fold of a 2-rank split of a periodic box
config4_helm3.npz  configs[4] in miniature: 3-component Helmholtz, N = 9,
                   2x2x2 elements, lam0 = 1/Re (Re = 1000), lam1 = beta0/dt
                   (11/6 / 1e-3), rhs default_rng(5 + c), Jacobi PCG tol 1e-6
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import gs as ogs  # noqa: E402
from oracle import mesh as om  # noqa: E402
from oracle import operators as oop  # noqa: E402
from oracle import partition as opart  # noqa: E402
from oracle import solvers as osol  # noqa: E402


def bp5_problem(o, lam0=1.0, lam1=0.0, rhs=None):
    mask = o.mask.ravel()
    D, G = o.basis.diff, o.G
    sh = (o.G.shape[0],) + o.G.shape[2:]
    if rhs is None:
        X = o.xyz.reshape(3, -1)
        rhs = o.B.ravel() * 3 * np.pi ** 2 * np.prod(np.sin(np.pi * X), axis=0)
    b = mask * ogs.gs_op(o.ids, rhs)

    def A(v):
        return mask * ogs.gs_op(o.ids, oop.bk5(D, G, v.reshape(sh), lam0=lam0, B=o.B,
                                               lam1=lam1).ravel())

    inv = mask / ogs.gs_op(o.ids, oop.local_diagonal(D, G, lam0, o.B, lam1).ravel())
    return b, A, inv, 1.0 / ogs.multiplicity(o.ids)


def config0():
    out = {}
    for tag, deform in (("deformed", ("sine", 0.05)), ("affine", None)):
        o = om.build_box_mesh((1.0, 1.0, 1.0), (4, 4, 4), 7, deformation=deform)
        b, A, inv, wt = bp5_problem(o)
        r = osol.pcg(A, lambda v: inv * v, b, tol=1e-8, max_iter=1000, weights=wt)
        out[f"{tag}_ids"] = o.ids.astype(np.int32)
        out[f"{tag}_mask"] = o.mask.astype(np.uint8)
        out[f"{tag}_b"] = b
        out[f"{tag}_x"] = r.x
        out[f"{tag}_iterations"] = np.int64(r.iterations)
        out[f"{tag}_history"] = np.asarray(r.residual_history)
    return out


def config1():
    out = {}
    for N, counts in ((3, (3, 3, 3)), (7, (2, 2, 2)), (11, (2, 1, 1)), (15, (2, 1, 1))):
        o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, deformation=("sine", 0.05))
        u = np.random.default_rng(1000 + N).standard_normal((o.E, N + 1, N + 1, N + 1))
        out[f"N{N}_counts"] = np.asarray(counts)
        out[f"N{N}_u"] = u
        out[f"N{N}_w"] = oop.bk5(o.basis.diff, o.G, u)
        if N == 7:
            out["N7_w_helmholtz"] = oop.bk5(o.basis.diff, o.G, u, lam0=0.25, B=o.B, lam1=3.0)
    return out


def config23():
    out = {}
    for tag, counts, P in (("c2", (64, 64, 64), 8), ("c3", (40, 20, 20), 2)):
        nx, ny, nz = counts
        el = np.arange(nx * ny * nz)
        cent = np.stack([el % nx, (el // nx) % ny, el // (nx * ny)], axis=1) + 0.5
        out[f"{tag}_part"] = opart.rcb(cent, P).astype(np.int8)
    # multi-rank canonical fold on a periodic box split over two ranks
    o = om.build_box_mesh((1.0, 1.0, 1.0), (4, 3, 2), 3, bc="periodic")
    nq3 = 64
    cent = o.xyz.reshape(3, o.E, nq3).mean(axis=2).T
    part = opart.rcb(cent, 2)
    rng = np.random.default_rng(2323)
    ids = [o.ids.reshape(o.E, nq3)[part == r].ravel() for r in range(2)]
    ws = [rng.standard_normal(len(i)) for i in ids]
    folded = ogs.gs_op_multi(ids, ws)
    out["gs_part"] = part.astype(np.int8)
    for r in range(2):
        out[f"gs_w{r}"] = ws[r]
        out[f"gs_out{r}"] = folded[r]
    return out


def config4():
    out = {}
    N, counts = 9, (2, 2, 2)
    lam0, lam1 = 1.0 / 1000.0, (11.0 / 6.0) / 1e-3
    o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, deformation=("sine", 0.05))
    for c in range(3):
        rhs = np.random.default_rng(5 + c).standard_normal(o.ids.size)
        b, A, inv, wt = bp5_problem(o, lam0, lam1, rhs=rhs)
        r = osol.pcg(A, lambda v: inv * v, b, tol=1e-6, max_iter=1000, weights=wt)
        out[f"b{c}"] = b
        out[f"x{c}"] = r.x
        out[f"iterations{c}"] = np.int64(r.iterations)
    out["lam"] = np.array([lam0, lam1])
    return out


def main():
    for name, fn in (("config0_bp5", config0), ("config1_bk5", config1),
                     ("config23_part", config23), ("config4_helm3", config4)):
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, **fn())
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
