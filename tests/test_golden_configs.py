"""The oracle reproduces the committed per-config golden fixtures
(tests/golden/make_config_golden.py) -- catches drift in the checker itself.
Integers (ids, masks, partitions, iteration counts) and the canonical gs fold
exactly; floating-point fields to 1e-13 relative (BLAS builds may differ in
the last bits of a matmul)."""

import os

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om
from oracle import operators as oop
from oracle import partition as opart
from oracle import solvers as osol

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(HERE, name + ".npz"))


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def _gen():
    import importlib.util
    spec = importlib.util.spec_from_file_location("mkg", os.path.join(HERE,
                                                                       "make_config_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("tag,deform", [("deformed", ("sine", 0.05)), ("affine", None)])
def test_config0_fixture(tag, deform):
    g = load("config0_bp5")
    o = om.build_box_mesh((1.0, 1.0, 1.0), (4, 4, 4), 7, deformation=deform)
    assert np.array_equal(o.ids.astype(np.int32), g[f"{tag}_ids"])
    assert np.array_equal(o.mask.astype(np.uint8), g[f"{tag}_mask"])
    b, A, inv, wt = _gen().bp5_problem(o)
    assert rel(b, g[f"{tag}_b"]) < 1e-13
    r = osol.pcg(A, lambda v: inv * v, b, tol=1e-8, max_iter=1000, weights=wt)
    assert r.iterations == int(g[f"{tag}_iterations"])
    assert rel(r.x, g[f"{tag}_x"]) < 1e-12


def test_config1_fixture():
    g = load("config1_bk5")
    for N in (3, 7, 11, 15):
        counts = tuple(int(c) for c in g[f"N{N}_counts"])
        o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, deformation=("sine", 0.05))
        u = np.random.default_rng(1000 + N).standard_normal((o.E, N + 1, N + 1, N + 1))
        assert np.array_equal(u, g[f"N{N}_u"])
        assert rel(oop.bk5(o.basis.diff, o.G, u), g[f"N{N}_w"]) < 1e-13
        if N == 7:
            assert rel(oop.bk5(o.basis.diff, o.G, u, lam0=0.25, B=o.B, lam1=3.0),
                       g["N7_w_helmholtz"]) < 1e-13


def test_config23_fixture():
    g = load("config23_part")
    for tag, counts, P in (("c2", (64, 64, 64), 8), ("c3", (40, 20, 20), 2)):
        nx, ny, nz = counts
        el = np.arange(nx * ny * nz)
        cent = np.stack([el % nx, (el // nx) % ny, el // (nx * ny)], axis=1) + 0.5
        part = opart.rcb(cent, P)
        assert np.array_equal(part.astype(np.int8), g[f"{tag}_part"])
        cnt = np.bincount(part, minlength=P)
        assert cnt.max() - cnt.min() <= 1
    o = om.build_box_mesh((1.0, 1.0, 1.0), (4, 3, 2), 3, bc="periodic")
    part = g["gs_part"].astype(np.int64)
    ids = [o.ids.reshape(o.E, 64)[part == r].ravel() for r in range(2)]
    out = ogs.gs_op_multi(ids, [g["gs_w0"], g["gs_w1"]])
    assert np.array_equal(out[0], g["gs_out0"]) and np.array_equal(out[1], g["gs_out1"])


def test_config4_fixture():
    g = load("config4_helm3")
    lam0, lam1 = g["lam"]
    o = om.build_box_mesh((1.0, 1.0, 1.0), (2, 2, 2), 9, deformation=("sine", 0.05))
    mk = _gen()
    for c in range(3):
        rhs = np.random.default_rng(5 + c).standard_normal(o.ids.size)
        b, A, inv, wt = mk.bp5_problem(o, lam0, lam1, rhs=rhs)
        assert rel(b, g[f"b{c}"]) < 1e-13
        r = osol.pcg(A, lambda v: inv * v, b, tol=1e-6, max_iter=1000, weights=wt)
        assert r.iterations == int(g[f"iterations{c}"])
        assert rel(r.x, g[f"x{c}"]) < 1e-12
