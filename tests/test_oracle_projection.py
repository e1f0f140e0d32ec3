"""CPU: the projection oracle (oracle/projection.py) against SPEC.md's
ProjectionSpace / project_guess / update examples."""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om
from oracle import operators as oop
from oracle import projection as oproj


@pytest.fixture(scope="module")
def problem():
    m = om.build_box_mesh((1, 1, 1), (2, 2, 2), 4, bc="dirichlet", deformation=("sine", 0.05))
    D, G = m.basis.diff, m.G
    mask = m.mask.ravel()
    shape = (m.E,) + (5,) * 3
    A = lambda v: mask * ogs.gs_op(m.ids, oop.bk5(D, G, v.reshape(shape)).ravel())
    inv = mask / ogs.gs_op(m.ids, oop.local_diagonal(D, G).ravel())
    M = lambda r: inv * r
    wt = 1.0 / ogs.multiplicity(m.ids)
    X = m.xyz.reshape(3, -1)
    f = 3 * np.pi ** 2 * np.prod(np.sin(np.pi * X), axis=0)
    b = mask * ogs.gs_op(m.ids, m.B.ravel() * f)
    # random-rhs variant and a next "time step" differing by 1%
    rng = np.random.default_rng(2104_05829)
    b = mask * ogs.gs_op(m.ids, m.B.ravel() * rng.standard_normal(mask.size))
    d = mask * ogs.gs_op(m.ids, m.B.ravel() * rng.standard_normal(mask.size))
    b2 = b + 0.01 * np.linalg.norm(b) / np.linalg.norm(d) * d
    return m, A, M, wt, b, mask, b2


def _rand(m, mask, seed):
    x = np.random.default_rng(seed).standard_normal(mask.size)
    return mask * ogs.gs_op(m.ids, x / ogs.multiplicity(m.ids))


def test_empty_space_zero_guess(problem):
    m, A, M, wt, b, mask, b2 = problem
    sp = oproj.ProjectionSpace(8, wt)
    x0, bd = sp.project(b)
    assert not np.any(x0) and np.array_equal(bd, b)


def test_same_rhs_twice_zero_iterations(problem):
    m, A, M, wt, b, mask, b2 = problem
    sp = oproj.ProjectionSpace(8, wt)
    r1 = oproj.solve_projected(sp, A, M, b, tol=1e-8)
    assert r1.converged and r1.iterations > 5
    r2 = oproj.solve_projected(sp, A, M, b, tol=1e-8)
    assert r2.iterations == 0 and r2.converged
    assert np.max(np.abs(r2.x - r1.x)) < 1e-8 * np.max(np.abs(r1.x))


def test_nearby_rhs_fewer_iterations(problem):
    m, A, M, wt, b, mask, b2 = problem
    sp = oproj.ProjectionSpace(8, wt)
    r1 = oproj.solve_projected(sp, A, M, b, tol=1e-8)
    assert abs(np.linalg.norm(b2 - b) / np.linalg.norm(b) - 0.01) < 1e-12
    r2 = oproj.solve_projected(sp, A, M, b2, tol=1e-8)
    plain = oproj.solve_projected(oproj.ProjectionSpace(8, wt), A, M, b2, tol=1e-8)
    assert r2.iterations < r1.iterations and r2.iterations < plain.iterations
    # same answer as the unprojected solve, to the tolerance
    assert np.linalg.norm(r2.x - plain.x) < 1e-6 * np.linalg.norm(plain.x)


def test_a_orthonormal_and_eviction(problem):
    m, A, M, wt, b, mask, b2 = problem
    sp = oproj.ProjectionSpace(3, wt)
    for s in range(5):
        x = _rand(m, mask, 10 + s)
        sp.update(x, A(x))
    assert sp.size == 3
    G = np.array([[sp.dot(xi, axj) for axj in sp.AX] for xi in sp.X])
    assert np.max(np.abs(G - np.eye(3))) < 1e-8
    # the newest solution lies in the span: projecting A x reproduces x
    x = _rand(m, mask, 14)
    x0, bd = sp.project(A(x))
    assert np.linalg.norm(x0 - x) < 1e-8 * np.linalg.norm(x)


def test_degenerate_update_restarts(problem):
    m, A, M, wt, b, mask, b2 = problem
    sp = oproj.ProjectionSpace(8, wt)
    x = _rand(m, mask, 5)
    y = _rand(m, mask, 6)
    sp.update(y, A(y))
    sp.update(x, A(x))
    assert sp.size == 2
    sp.update(x, A(x))            # already in the span -> restart with x only
    assert sp.size == 1
    assert abs(sp.dot(sp.X[0], sp.AX[0]) - 1.0) < 1e-12
    sp.update(0 * x, 0 * x)       # zero solution is ignored
    assert sp.size == 1
