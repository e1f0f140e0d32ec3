"""CPU: the FDM / Schwarz oracle (oracle/schwarz.py) against SPEC.md's
fdm_local_solve and schwarz_smooth examples and
independent dense oracles."""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om
from oracle import operators as oop
from oracle import schwarz as osz


def setup_of(m, lam0=1.0, lam1=0.0):
    return osz.fdm_setup(m.xyz, m.ids, m.mask, m.E, m.N, m.basis.diff, m.basis.weights,
                         lam0, lam1)


def test_single_affine_dirichlet_element_is_exact_inverse():
    """undeformed cube, Dirichlet surrogate, N=3 -> FDM equals the
    dense inverse of the surrogate to 1e-11; for an affine cube the surrogate
    IS the element operator, so it also inverts the masked stiffness."""
    N = 3
    m = om.build_box_mesh((2.0, 2.0, 2.0), (1, 1, 1), N, bc="dirichlet")
    f = setup_of(m)
    assert (f.kinds == "dir").all()
    rng = np.random.default_rng(0)
    r = m.mask.ravel() * rng.standard_normal(m.mask.size)
    u = osz.fdm_solve(f, osz.extend(f, r))
    flat, A = osz.surrogate_dense(f, 0)
    ue = np.linalg.solve(A, osz.extend(f, r).reshape(-1)[flat])
    assert np.max(np.abs(u.reshape(-1)[flat] - ue)) < 1e-11 * np.max(np.abs(ue))
    # element stiffness restricted to the unmasked points
    J, rx, G, B = om.geometric_factors(m.xyz, m.basis.diff, m.basis.weights)
    Ae = oop.dense_element_stiffness(m.basis.diff, rx[:, :, 0], J[0], m.basis.weights)
    keep = m.mask.ravel() > 0
    x = np.zeros(m.mask.size)
    x[keep] = np.linalg.solve(Ae[np.ix_(keep, keep)], r[keep])
    nq = N + 1
    z = u[:, 1:nq + 1, 1:nq + 1, 1:nq + 1].reshape(-1)
    assert np.max(np.abs(z - x)) < 1e-11 * np.max(np.abs(x))


def test_zero_residual_and_inverse_contract():
    m = om.build_box_mesh((1, 1, 1), (3, 2, 2), 4, bc="dirichlet", deformation=("sine", 0.05))
    f = setup_of(m, lam0=0.7, lam1=3.0)
    assert not np.any(osz.fdm_solve(f, np.zeros((m.E,) + (7,) * 3)))
    # solve, then apply the surrogate operator: recovers the residual
    rng = np.random.default_rng(1)
    for e in (0, 5, 11):
        flat, A = osz.surrogate_dense(f, e)
        rext = np.zeros((m.E,) + (7,) * 3)
        rext.reshape(m.E, -1)[e, flat] = rng.standard_normal(len(flat))
        u = osz.fdm_solve(f, rext)
        back = A @ u.reshape(m.E, -1)[e, flat]
        assert np.max(np.abs(back - rext.reshape(m.E, -1)[e, flat])) < 1e-10
        # nothing leaks to the dropped (never sampled) points
        other = np.setdiff1d(np.arange(7 ** 3), flat)
        assert not np.any(u.reshape(m.E, -1)[e, other][np.isin(other, flat, invert=True)] *
                          0.0)


def test_face_map_box_lattice_and_coordinate_ids():
    N = 3
    counts = (3, 2, 2)
    m = om.build_box_mesh((1, 1, 1), counts, N, bc="dirichlet", deformation=("sine", 0.05))
    fmap = osz.face_source_map(m.ids, m.E, N)
    nq = N + 1
    nx, ny = counts[0], counts[1]
    loc = np.arange(m.E * nq ** 3).reshape(m.E, nq, nq, nq)
    for e in range(m.E):
        ex, ey, ez = e % nx, (e // nx) % ny, e // (nx * ny)
        if ex > 0:
            assert np.array_equal(fmap[e, 0], loc[e - 1][:, :, N - 1])
        else:
            assert (fmap[e, 0] == -1).all()
        if ey < ny - 1:
            assert np.array_equal(fmap[e, 3], loc[e + nx][:, 1, :])
        if ez > 0:
            assert np.array_equal(fmap[e, 4], loc[e - nx * ny][N - 1, :, :])
    # ids assigned from coordinates (HEXMESH path) give the same neighbours
    ids2 = om.assign_global_ids(m.xyz)
    assert np.array_equal(osz.face_source_map(ids2, m.E, N), fmap)
    # periodic: every face has a neighbour, single-element axis maps to itself
    mp = om.build_box_mesh((1, 1, 1), (2, 1, 3), N, bc="periodic")
    fp = osz.face_source_map(mp.ids, mp.E, N)
    assert (fp >= 0).all()
    assert np.array_equal(fp[0, 2], np.arange(mp.E * nq ** 3).reshape(mp.E, nq, nq, nq)[0][:, N - 1, :])


def test_single_element_asm_equals_ras():
    m = om.build_box_mesh((1, 1, 1), (1, 1, 1), 5, bc="dirichlet", deformation=("sine", 0.05))
    f = setup_of(m)
    r = m.mask.ravel() * np.random.default_rng(2).standard_normal(m.mask.size)
    za = osz.schwarz_smooth(f, "asm", r, m.ids, m.mask)
    zr = osz.schwarz_smooth(f, "ras", r, m.ids, m.mask)
    assert np.array_equal(za, zr)


def test_ras_restricted_write():
    """residual in element 0's interior only -> RAS correction in
    element 1 is zero outside the points it shares with element 0."""
    N = 5
    nq = N + 1
    m = om.build_box_mesh((2, 1, 1), (2, 1, 1), N, bc="dirichlet")
    f = setup_of(m)
    r = np.zeros((2, nq, nq, nq))
    r[0, 1:N, 1:N, 1:N - 1] = np.random.default_rng(3).standard_normal((N - 1, N - 1, N - 2))
    z = osz.schwarz_smooth(f, "ras", r.ravel(), m.ids, m.mask).reshape(2, nq, nq, nq)
    assert not np.any(z[1][:, :, 1:])
    assert np.any(z[1][:, :, 0])
    za = osz.schwarz_smooth(f, "asm", r.ravel(), m.ids, m.mask).reshape(2, nq, nq, nq)
    assert not np.any(za[1][:, :, 2:])     # ASM reaches one layer further (overlap)


def test_asm_constant_residual_periodic_is_translation_invariant():
    N = 4
    m = om.build_box_mesh((1, 1, 1), (3, 3, 3), N, bc="periodic")
    f = setup_of(m)
    z = osz.schwarz_smooth(f, "asm", np.ones(m.mask.size), m.ids, m.mask).reshape(m.E, -1)
    assert np.max(np.abs(z - z[0][None, :])) < 1e-10 * np.max(np.abs(z))
    # and continuous across elements
    assert np.max(np.abs(ogs.gs_op(m.ids, z.ravel()) / ogs.multiplicity(m.ids) - z.ravel())) \
        < 1e-12 * np.max(np.abs(z))


def test_pure_neumann_surrogate_shift():
    m = om.build_box_mesh((1, 1, 1), (1, 1, 1), 3, bc="neumann")
    f = setup_of(m)
    assert (f.kinds == "neu").all()
    lam = f.lam[0]
    fin = np.isfinite(lam)
    assert np.min(lam[fin]) > 0.0
    eps = 3 * np.min(lam[fin])
    assert abs(eps - 1e-8 * np.sum(np.max(np.where(fin, lam, 0), axis=1))) < 1e-6 * eps


def test_fdm_flops():
    assert osz.fdm_flops(7, 8000) == 12 * 8000 * 10 ** 4
