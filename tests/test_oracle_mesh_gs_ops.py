"""SPEC known-answer tests that pin the oracle's mesh, gs, operators, PCG and
RCB (no reference implementation of these exists)."""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om
from oracle import operators as oop
from oracle import partition as opart
from oracle import solvers as osol


# ------------------------------------------------------------------ mesh
def test_single_cube_side_two():
    m = om.build_box_mesh((2, 2, 2), (1, 1, 1), 1, bc="neumann", origin=(-1, -1, -1))
    assert m.xyz.shape == (3, 1, 2, 2, 2)
    assert np.allclose(m.J, 1.0)
    assert np.allclose(m.G[:, [1, 2, 4]], 0.0)
    w = m.basis.weights
    rho = w[:, None, None] * w[None, :, None] * w[None, None, :]
    for c in (0, 3, 5):
        assert np.allclose(m.G[0, c], rho)


def test_scaled_element_factors():
    a = om.build_box_mesh((2, 2, 2), (1, 1, 1), 3, bc="neumann")
    b = om.build_box_mesh((4, 2, 2), (1, 1, 1), 3, bc="neumann")
    assert np.allclose(b.J, 2 * a.J)
    assert np.allclose(b.G[:, 0], 0.5 * a.G[:, 0])
    assert np.allclose(b.G[:, 3], 2 * a.G[:, 3])
    assert np.allclose(b.G[:, 5], 2 * a.G[:, 5])


def test_volume_and_deformed_volume():
    m = om.build_box_mesh((1, 2, 3), (3, 2, 2), 4, bc="neumann")
    assert abs(m.B.sum() - 6.0) < 1e-12
    d = om.build_box_mesh((1, 1, 1), (4, 4, 4), 7, deformation=("sine", 0.05))
    assert np.all(d.J > 0)
    assert abs(d.B.sum() - 1.0) < 1e-10           # boundary-preserving map


def test_shared_face_ids():
    m = om.build_box_mesh((2, 1, 1), (2, 1, 1), 1, bc="neumann")
    ids = m.ids.reshape(2, 2, 2, 2)
    assert np.array_equal(ids[0, :, :, 1], ids[1, :, :, 0])
    z = om.singleton_ids(m.ids)
    nz = z[z != 0]
    assert len(np.unique(nz)) == 4
    assert all(np.sum(z == g) == 2 for g in np.unique(nz))
    one = om.build_box_mesh((1, 1, 1), (1, 1, 1), 3, bc="neumann")
    assert np.all(om.singleton_ids(one.ids) == 0)


def test_periodic_id_count():
    m = om.build_box_mesh((1, 1, 1), (4, 4, 4), 7, bc="periodic")
    assert len(np.unique(m.ids)) == 28 ** 3 == 21952


def test_ids_match_coordinate_sort():
    m = om.build_box_mesh((1, 1, 1), (3, 2, 2), 3, bc="dirichlet")
    ids2 = om.assign_global_ids(m.xyz.reshape(3, -1))
    assert np.array_equal(ids2, m.ids)
    # shuffled element order -> same multiset of (coordinate -> id)
    perm = np.random.default_rng(5).permutation(m.E)
    xs = m.xyz[:, perm].reshape(3, -1)
    ids3 = om.assign_global_ids(xs)
    assert np.array_equal(ids3, m.ids.reshape(m.E, -1)[perm].ravel())


def test_box_unique_counts():
    m = om.build_box_mesh((1, 1, 1), (20, 20, 20), 7, bc="dirichlet")
    assert m.ids.max() == 141 ** 3 == 2803221


def test_hexmesh_roundtrip(tmp_path):
    m = om.build_box_mesh((1, 1, 1), (2, 1, 1), 2, deformation=("sine", 0.05))
    p = tmp_path / "m.hex"
    om.write_hexmesh(p, m.xyz, m.ids, {"pressure": m.mask.astype(int)})
    E, N, xyz, ids, masks = om.read_hexmesh(p)
    assert (E, N) == (2, 2)
    assert np.array_equal(xyz, m.xyz) and np.array_equal(ids, m.ids)
    assert np.array_equal(masks["pressure"], m.mask.astype(int).ravel())


# ------------------------------------------------------------------ gs
def test_gs_examples():
    assert np.array_equal(ogs.gs_op([5, 5], [3.5, 3.5]), [7.0, 7.0])
    assert np.array_equal(ogs.gs_op([2, 2, 2], [2.0, 5.0, -1.0], "min"), [-1, -1, -1])
    assert np.array_equal(ogs.gs_op([2, 2, 2], [2.0, 5.0, -1.0], "max"), [5, 5, 5])
    assert np.array_equal(ogs.gs_op([0, 0, 0], [1.0, 2.0, 3.0]), [1, 2, 3])
    with pytest.raises(ValueError):
        ogs.gs_op([1, 1], [1.0, 2.0, 3.0])


def test_gs_two_rank_toy():
    out = ogs.gs_op_multi([np.array([0, 7, 0]), np.array([7, 0, 0])],
                          [np.array([1.0, 2.0, 3.0]), np.array([10.0, 20.0, 30.0])])
    assert np.array_equal(out[0], [1, 12, 3]) and np.array_equal(out[1], [12, 20, 30])


@pytest.mark.parametrize("seed", range(20))
def test_gs_vs_dense_Q(seed):
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, 40, size=200)
    w = rng.standard_normal(200)
    Q = ogs.dense_Q(ids)
    ref = Q @ (Q.T @ w)
    assert np.allclose(ogs.gs_op(ids, w), ref, rtol=0, atol=1e-13)


def test_gs_projection_property():
    m = om.build_box_mesh((1, 1, 1), (3, 3, 3), 3, bc="neumann")
    rng = np.random.default_rng(1)
    w = rng.standard_normal(m.ids.size)
    inv = 1.0 / ogs.multiplicity(m.ids)
    once = inv * ogs.gs_op(m.ids, w)
    twice = inv * ogs.gs_op(m.ids, once)
    assert np.allclose(once, twice, atol=1e-14)


# ------------------------------------------------------------------ operators
def _dense(m):
    D, w = m.basis.diff, m.basis.weights
    blocks = []
    for e in range(m.E):
        J, rx, G, B = om.geometric_factors(m.xyz[:, e:e + 1], D, w)
        blocks.append(oop.dense_element_stiffness(D, rx[:, :, 0], J[0], w))
    return blocks


@pytest.mark.parametrize("N,counts,deform", [(2, (2, 1, 1), None), (3, (1, 1, 3), ("sine", 0.05)),
                                             (2, (2, 1, 1), ("sine", 0.08))])
def test_bk5_vs_dense_assembly(N, counts, deform):
    m = om.build_box_mesh((1, 1, 1), counts, N, bc="neumann", deformation=deform)
    blocks = _dense(m)
    Q, A, AL = oop.dense_assembled(m.ids, blocks)
    rng = np.random.default_rng(N)
    uL = rng.standard_normal(m.ids.size)
    wmf = oop.bk5(m.basis.diff, m.G, uL.reshape(m.E, N + 1, N + 1, N + 1))
    assert np.max(np.abs(AL @ uL - wmf.ravel())) < 1e-12 * max(1, np.abs(AL).max())
    assert np.max(np.abs(A @ np.ones(A.shape[0]))) < 1e-12      # Neumann nullspace
    assert np.max(np.abs(A - A.T)) < 1e-12                      # symmetry
    dg = oop.local_diagonal(m.basis.diff, m.G)
    assert np.max(np.abs(np.diag(AL) - dg.ravel())) < 1e-12
    dga = ogs.gs_op(m.ids, dg.ravel())
    assert np.allclose(dga, (Q @ np.diag(A)), atol=1e-12)


def test_helmholtz_and_mass():
    m = om.build_box_mesh((1, 1, 1), (2, 2, 1), 3, bc="neumann", deformation=("sine", 0.05))
    rng = np.random.default_rng(3)
    u = rng.standard_normal((m.E, 4, 4, 4))
    w = oop.bk5(m.basis.diff, m.G, u, lam0=0.3, B=m.B, lam1=7.0)
    w_ref = 0.3 * oop.bk5(m.basis.diff, m.G, u) + 7.0 * m.B * u
    assert np.allclose(w, w_ref, rtol=1e-14, atol=1e-14)
    a = om.build_box_mesh((1, 1, 1), (2, 2, 1), 3, bc="neumann")
    one = np.ones_like(u)
    assert abs(oop.inner_product(a.B, one, one) - 1.0) < 1e-12
    s1 = om.build_box_mesh((2, 2, 2), (1, 1, 1), 2, bc="neumann", origin=(-1, -1, -1))
    x = s1.xyz[0]
    assert abs(oop.inner_product(s1.B, x, x) - 8.0 / 3.0) < 1e-12
    d = oop.local_diagonal(m.basis.diff, m.G, lam0=1.0, B=m.B, lam1=1e12)
    assert np.allclose(d / (1e12 * m.B), 1.0, rtol=1e-6)


def test_flop_counter_formula():
    assert oop.bk5_flops(7, 1) == 12 * 8 ** 4 + 15 * 8 ** 3 == 56832
    assert oop.bk5_memrefs(7, 8000) == 7 * 8000 * 512


# ------------------------------------------------------------------ pcg
def test_pcg_examples():
    r = osol.pcg(lambda v: v, lambda v: v, np.zeros(4))
    assert r.iterations == 0 and np.all(r.x == 0)
    d = np.array([1.0, 2.0, 3.0])
    r = osol.pcg(lambda v: d * v, lambda v: v / d, np.array([1.0, 1.0, 1.0]), tol=1e-12)
    assert r.iterations == 1 and np.allclose(r.x, 1 / d)
    with pytest.raises(osol.BreakdownError):
        osol.pcg(lambda v: -v, lambda v: v, np.ones(3))


def test_pcg_poisson_vs_dense():
    m = om.build_box_mesh((1, 1, 1), (2, 2, 2), 4, bc="dirichlet")
    blocks = _dense(m)
    Q, A, AL = oop.dense_assembled(m.ids, blocks)
    mask = m.mask.ravel()
    mult = ogs.multiplicity(m.ids)
    X = m.xyz.reshape(3, -1)
    f = 3 * np.pi ** 2 * np.prod(np.sin(np.pi * X), axis=0)
    b = mask * ogs.gs_op(m.ids, m.B.ravel() * f)
    D, G = m.basis.diff, m.G
    sh = (m.E, 5, 5, 5)

    def A_op(v):
        return mask * ogs.gs_op(m.ids, oop.bk5(D, G, v.reshape(sh)).ravel())

    diag = ogs.gs_op(m.ids, oop.local_diagonal(D, G).ravel())
    inv = mask / diag
    res = osol.pcg(A_op, lambda r: inv * r, b, tol=1e-8, max_iter=500, weights=1 / mult)
    assert res.converged
    # dense direct solve on the unmasked unique dofs
    maskg = (Q.T @ mask) / (Q.T @ np.ones_like(mask)) > 0.5
    bg = (Q.T @ (b / mult))
    xg = np.zeros(Q.shape[1])
    xg[maskg] = np.linalg.solve(A[np.ix_(maskg, maskg)], bg[maskg])
    assert np.max(np.abs(Q @ xg - res.x)) < 1e-7
    # flexible with a fixed SPD preconditioner gives the same iterates
    res2 = osol.pcg(A_op, lambda r: inv * r, b, tol=1e-8, max_iter=500, weights=1 / mult,
                    flexible=True)
    assert abs(res2.iterations - res.iterations) <= 1
    assert np.max(np.abs(res2.x - res.x)) < 1e-7


# ------------------------------------------------------------------ rcb
def test_rcb_examples():
    line = np.c_[np.arange(8.0), np.zeros(8), np.zeros(8)]
    assert list(opart.rcb(line, 2)) == [0, 0, 0, 0, 1, 1, 1, 1]
    assert np.all(opart.rcb(line, 1) == 0)
    g = np.array([[x, y, 0.0] for y in range(4) for x in range(4)])
    p = opart.rcb(g, 4)
    for r in range(4):
        pts = g[p == r]
        assert len(pts) == 4
        assert np.ptp(pts[:, 0]) == 1 and np.ptp(pts[:, 1]) == 1


@pytest.mark.parametrize("E,P", [(5, 2), (7, 4), (100, 8), (64, 3), (1000, 7)])
def test_rcb_balance(E, P):
    rng = np.random.default_rng(E + P)
    p = opart.rcb(rng.random((E, 3)), P)
    cnt = np.bincount(p, minlength=P)
    assert cnt.max() - cnt.min() <= 1
