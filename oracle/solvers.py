"""Oracle: preconditioned conjugate gradients.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates SPEC.md:479-487:
  * stop when ||r||_2 <= tol * ||b||_2 (plain 2-norm of the assembled
    residual; on L-vectors that is sqrt(sum_L r^2 / mult));
  * b = 0 -> x = 0 in 0 iterations;
  * p^T A p <= 0 -> breakdown error;
  * max_iter exceeded -> last iterate with converged=False;
  * Fletcher-Reeves beta (standard) or Polak-Ribiere beta
    z_k^T (r_k - r_{k-1}) / z_{k-1}^T r_{k-1} (flexible).
Iteration structure (SURVEY.md §3 call stack 4): Ap, alpha, x/r update,
convergence check, z = M r, beta, p update.
"""

from collections import namedtuple

import numpy as np

PCGResult = namedtuple("PCGResult", "x iterations residual_history converged")


class BreakdownError(RuntimeError):
    pass


def pcg(apply_A, apply_M, b, tol=1e-8, max_iter=1000, flexible=False, weights=None,
        x0=None):
    b = np.asarray(b, dtype=np.float64)
    wt = np.ones_like(b) if weights is None else np.asarray(weights, dtype=np.float64)

    def dot(a, c):
        return float(np.sum(wt * a * c))

    bnorm = np.sqrt(dot(b, b))
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    if bnorm == 0.0:
        return PCGResult(np.zeros_like(b), 0, [0.0], True)
    r = b - apply_A(x) if x0 is not None else b.copy()
    rnorm = np.sqrt(dot(r, r))
    hist = [rnorm]
    if rnorm <= tol * bnorm:
        return PCGResult(x, 0, hist, True)
    z = apply_M(r)
    p = z.copy()
    rz = dot(r, z)
    for k in range(max_iter):
        Ap = apply_A(p)
        pAp = dot(p, Ap)
        if not pAp > 0.0:
            raise BreakdownError(f"p^T A p = {pAp} <= 0 at iteration {k}")
        alpha = rz / pAp
        x += alpha * p
        r_old = r.copy() if flexible else None
        r -= alpha * Ap
        rnorm = np.sqrt(dot(r, r))
        hist.append(rnorm)
        if rnorm <= tol * bnorm:
            return PCGResult(x, k + 1, hist, True)
        z = apply_M(r)
        rz_new = dot(r, z)
        if flexible:
            beta = (rz_new - dot(z, r_old)) / rz
        else:
            beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    return PCGResult(x, max_iter, hist, False)
