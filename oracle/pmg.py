"""Oracle: Chebyshev-Jacobi smoothing and the p-multigrid V-cycle preconditioner.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates SPEC.md:466-471 (MultigridHierarchy), 489-497 (chebyshev_smooth),
509-517 (pmg_preconditioner), 519-527 (coarse_solve), 546-551 (design
decisions: multiplicative V-cycle, Chebyshev degree 2 with bounds 0.1-1.1 of
the estimated lambda_max, masking after every smoother application and
transfer).  Deviation: lambda_max from 20 power iterations
from a fixed-seed random start (power_lambda_max) instead of SPEC's 10 from
the ones vector.

Frozen choices:
  * levels: orders N, max(N//2, 1), 1 (deduplicated), same elements and the
    same box map evaluated at each order's GLL points;
  * transfers: prolongation e_f = (J x J x J) e_c per element with
    J = interp_matrix(coarse nodes -> fine nodes) (basis.py:99-117);
    restriction r_c = mask_c * QQ^T_c (J^T x J^T x J^T)(r_f / mult_f);
  * smoother: Chebyshev on S A with x0 = 0 (Saad's 3-term recurrence),
    `degree` terms, degree - 1 operator applications, S the inner smoother:
    D^-1 (cheby_jac; 'jacobi' = degree 1, the Chebyshev-optimal damped
    Jacobi), or an overlapping Schwarz solve (cheby_asm / cheby_ras,
    oracle/schwarz.py, PAPER.md:298-313 CHEBY-ASM); 'asm' / 'ras' apply the
    Schwarz smoother once, undamped;
  * V-cycle: pre-smooth, residual, restrict, recurse, prolong + correct,
    post-smooth on the updated residual; coarsest level: exact solve of the
    assembled masked operator (dense inverse on unique unmasked dofs).
  * Chebyshev bounds: SPEC.md:548's (0.1, 1.1) x lambda_max for cheby_jac;
    (0.4, 1.1) for cheby_asm / cheby_ras.  Deviation: with 0.1 the degree-2
    polynomial damps the whole S A spectrum by ~0.53, worse than one
    undamped Schwarz application (lambda_max(S A) ~ 1.5), so CHEBY-ASM took
    10 iterations vs ASM's 7 on SPEC.md:541's problem; 0.4 gives 5
    (profiles/r2_smoother_bounds.jsonl).
"""

import numpy as np

from . import gs as ogs
from . import mesh as om
from . import operators as oop
from . import schwarz as osz
from .basis import Basis, interp_matrix

SMOOTHERS = ("jacobi", "cheby_jac", "asm", "ras", "cheby_asm", "cheby_ras")


class Level:
    pass


def orders_for(N):
    out = []
    for n in (N, max(N // 2, 1), 1):
        if n not in out:
            out.append(n)
    return out


def _apply_op(lv, v):
    sh = (lv.mesh.E,) + (lv.nq,) * 3
    return lv.mask * ogs.gs_op(lv.mesh.ids, oop.bk5(lv.mesh.basis.diff, lv.mesh.G,
                                                    v.reshape(sh), lv.lam0, lv.mesh.B,
                                                    lv.lam1).ravel())


def _interp3(M, v, E):
    """out[e] = (M x M x M) v[e]; M (no, ni); v (E, ni, ni, ni) [k][j][i]."""
    ni = M.shape[1]
    v = v.reshape(E, ni, ni, ni)
    t = np.einsum("ai,ekji->ekja", M, v)
    t = np.einsum("bj,ekja->ekba", M, t)
    t = np.einsum("ck,ekba->ecba", M, t)
    return t


def inner(lv, r):
    """The inner smoother S r of a level (D^-1, or Schwarz)."""
    if lv.schwarz is None:
        return lv.invD * r
    return osz.schwarz_smooth(lv.fdm, lv.schwarz, r, lv.mesh.ids, lv.mask)


def power_lambda_max(lv, iters=20, seed=2104):
    """lambda_max of S A by power iteration.  Start vector: a fixed-seed
    random, assembled, masked field -- SPEC.md:491's masked ones vector is
    nearly free of high-frequency content and underestimates lambda_max by
    ~30% at N = 7 (10 iterations: 1.62 vs 2.41), which makes the Chebyshev
    smoother amplify the top of the spectrum."""
    x = np.random.default_rng(seed).standard_normal(lv.mask.size)
    x = lv.mask * ogs.gs_op(lv.mesh.ids, lv.wt * x)
    lam = 0.0
    for _ in range(iters):
        y = inner(lv, _apply_op(lv, x))
        lam = float(np.sqrt(np.sum(lv.wt * y * y)) / np.sqrt(np.sum(lv.wt * x * x)))
        x = y / np.sqrt(np.sum(lv.wt * y * y))
    return lam


def chebyshev_smooth(lv, r, degree, lo, hi):
    """Chebyshev-accelerated inner smoother on A e = r from e0 = 0
    (SPEC.md:489-497)."""
    theta = 0.5 * (hi + lo)
    delta = 0.5 * (hi - lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    res = r.copy()
    d = (1.0 / theta) * inner(lv, res)
    x = d.copy()
    for _ in range(1, degree):
        res = res - _apply_op(lv, d)
        rho_new = 1.0 / (2.0 * sigma - rho)
        d = (rho_new * rho) * d + (2.0 * rho_new / delta) * inner(lv, res)
        rho = rho_new
        x = x + d
    return x


def smooth(lv, r, degree):
    """One smoothing of A e = r from e0 = 0 with the level's smoother kind."""
    if lv.kind in ("asm", "ras"):
        return inner(lv, r)
    return chebyshev_smooth(lv, r, 1 if lv.kind == "jacobi" else degree, lv.lo, lv.hi)


def build_hierarchy(extent, counts, N, bc="dirichlet", deformation=None, lam0=1.0, lam1=0.0,
                    degree=2, bounds=None, power_iters=20, smoother="cheby_jac"):
    if smoother not in SMOOTHERS:
        raise ValueError(f"unknown smoother {smoother!r}")
    if bounds is None:        # (0.4, 1.1) for Chebyshev-Schwarz: see the module doc
        bounds = (0.4, 1.1) if smoother in ("cheby_asm", "cheby_ras") else (0.1, 1.1)
    levels = []
    for n in orders_for(N):
        lv = Level()
        lv.order, lv.nq = n, n + 1
        lv.mesh = om.build_box_mesh(extent, counts, n, bc=bc, deformation=deformation)
        lv.lam0, lv.lam1 = lam0, lam1
        lv.mask = lv.mesh.mask.ravel()
        lv.wt = 1.0 / ogs.multiplicity(lv.mesh.ids)
        diag = ogs.gs_op(lv.mesh.ids, oop.local_diagonal(lv.mesh.basis.diff, lv.mesh.G, lam0,
                                                         lv.mesh.B, lam1).ravel())
        lv.invD = lv.mask / diag
        lv.kind = smoother
        lv.schwarz = {"asm": "asm", "cheby_asm": "asm", "ras": "ras",
                      "cheby_ras": "ras"}.get(smoother)
        lv.fdm = None
        if lv.schwarz is not None and n != orders_for(N)[-1]:
            lv.fdm = osz.fdm_setup(lv.mesh.xyz, lv.mesh.ids, lv.mask, lv.mesh.E, n,
                                   lv.mesh.basis.diff, lv.mesh.basis.weights, lam0, lam1)
        levels.append(lv)
    for lv in levels[:-1]:
        lv.lmax = power_lambda_max(lv, power_iters)
        lv.lo, lv.hi = bounds[0] * lv.lmax, bounds[1] * lv.lmax
    for f, c in zip(levels[:-1], levels[1:]):
        f.J = interp_matrix(Basis.get(c.order).nodes, Basis.get(f.order).nodes)  # (nq_f, nq_c)
    levels[-1].coarse = _coarse_factor(levels[-1])
    return {"levels": levels, "degree": degree}


def _coarse_factor(lv):
    """Dense inverse of the assembled, masked coarse operator on the unique
    unmasked dofs, from dense element matrices."""
    m = lv.mesh
    D, w = m.basis.diff, m.basis.weights
    blocks = []
    for e in range(m.E):
        J, rx, G, B = om.geometric_factors(m.xyz[:, e:e + 1], D, w)
        Ae = oop.dense_element_stiffness(D, rx[:, :, 0], J[0], w) * lv.lam0
        if lv.lam1:
            Ae = Ae + lv.lam1 * np.diag(B[0].ravel())
        blocks.append(Ae)
    Q, A, AL = oop.dense_assembled(m.ids, blocks)
    keep = (Q.T @ lv.mask) > 0.5 * (Q.T @ np.ones_like(lv.mask))
    Ak = A[np.ix_(keep, keep)]
    # pure Neumann / periodic, no mass term: pin the constant,
    # pinv(A) = (A + 1 1^T)^-1 - 1 1^T / n^2 on the range of A
    singular = bool(keep.all()) and not lv.lam1
    nk_ = int(keep.sum())
    Ainv = np.zeros_like(A)
    if singular:
        Ainv[np.ix_(keep, keep)] = np.linalg.inv(Ak + 1.0) - 1.0 / nk_ ** 2
    else:
        Ainv[np.ix_(keep, keep)] = np.linalg.inv(Ak)
    # L-vector form: e_L = Q Ainv Q^T (r_L / mult)
    return Q, Ainv


def vcycle(h, r, level=0):
    """z = M^-1 r, one V-cycle."""
    L = h["levels"]
    lv = L[level]
    if level == len(L) - 1:
        Q, Ainv = lv.coarse
        return lv.mask * (Q @ (Ainv @ (Q.T @ (lv.wt * r))))
    deg = h["degree"]
    e = smooth(lv, r, deg)
    res = r - _apply_op(lv, e)
    c = L[level + 1]
    Jt = lv.J.T
    rc = _interp3(Jt, lv.wt * res, lv.mesh.E).ravel()
    rc = c.mask * ogs.gs_op(c.mesh.ids, rc)
    ec = vcycle(h, rc, level + 1)
    e = e + lv.mask * _interp3(lv.J, ec, lv.mesh.E).ravel()
    res = r - _apply_op(lv, e)
    e = e + smooth(lv, res, deg)
    return e


def fine_operator(h):
    lv = h["levels"][0]
    return lambda v: _apply_op(lv, v)
