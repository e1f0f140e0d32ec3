"""Oracle: projection-based initial guesses.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates SPEC.md:529-537 (ProjectionSpace, project_guess, update; PAPER.md:
250-251 "projection-based initial guesses", 323):
  * the space stores up to `capacity` (default 8) prior solutions x_i,
    A-orthonormal (x_i^T A x_j = delta_ij), and A x_i;
  * project: x0 = sum_i (x_i^T b) x_i, deflated rhs b' = b - A x0
    = b - sum_i (x_i^T b) A x_i; the solver then solves A dx = b';
  * update(x_new): when the space is full, evict the oldest first; then
    A-orthonormalise the new total solution against the remaining basis
    (classical Gram-Schmidt applied twice) and append it, so x_new always lies
    in the span afterwards; restart (clear, keep only x_new) when
    ||candidate||_A < 1e-10 ||x_new||_A.
Inner products are over unique dofs: <a, b> = sum_L a_L b_L / mult_L on
assembled L-vectors (the same convention as oracle/solvers.py).

Frozen choice: the solve after projection stops at
||b - A x|| <= tol ||b|| of the ORIGINAL rhs, i.e. the inner solver runs at
tol * ||b|| / ||b'||, and 0 iterations when ||b'|| <= tol ||b||.
"""

import numpy as np

from .solvers import PCGResult, pcg

DEGENERATE = 1e-10


class ProjectionSpace:
    def __init__(self, capacity=8, weights=None):
        if capacity < 1:
            raise ValueError("projection capacity must be >= 1")
        self.capacity = int(capacity)
        self.wt = weights
        self.X, self.AX = [], []

    def dot(self, a, b):
        return float(np.sum(a * b)) if self.wt is None else float(np.sum(self.wt * a * b))

    @property
    def size(self):
        return len(self.X)

    def clear(self):
        self.X, self.AX = [], []

    def project(self, b):
        x0 = np.zeros_like(b)
        bd = b.copy()
        for x, ax in zip(self.X, self.AX):
            c = self.dot(x, b)
            x0 += c * x
            bd -= c * ax
        return x0, bd

    def update(self, x_new, Ax_new):
        if len(self.X) >= self.capacity:        # evict the oldest
            self.X.pop(0)
            self.AX.pop(0)
        n0 = self.dot(x_new, Ax_new)
        if not n0 > 0.0:                        # zero solution: nothing to add
            return
        x, ax = x_new.copy(), Ax_new.copy()
        for _ in range(2):                      # CGS2
            cs = [self.dot(xi, ax) for xi in self.X]
            for c, xi, axi in zip(cs, self.X, self.AX):
                x -= c * xi
                ax -= c * axi
        n2 = self.dot(x, ax)
        if not n2 > (DEGENERATE ** 2) * n0:
            self.clear()
            x, ax, n2 = x_new.copy(), Ax_new.copy(), n0
        s = 1.0 / np.sqrt(n2)
        self.X.append(x * s)
        self.AX.append(ax * s)


def project_guess(space, b):
    return space.project(b)


def solve_projected(space, apply_A, apply_M, b, tol=1e-8, max_iter=1000, flexible=False):
    """x0, b' = project(b); PCG on A dx = b' to tol*||b||; x = x0 + dx;
    update(x).  Returns PCGResult with the inner iteration count."""
    wt = space.wt
    nb = np.sqrt(space.dot(b, b))
    x0, bd = space.project(b)
    nd = np.sqrt(space.dot(bd, bd))
    if nb == 0.0 or nd <= tol * nb:
        res = PCGResult(x0, 0, [nd], True)
    else:
        r = pcg(apply_A, apply_M, bd, tol=tol * nb / nd, max_iter=max_iter, flexible=flexible,
                weights=wt)
        res = r._replace(x=x0 + r.x)
    space.update(res.x, apply_A(res.x))
    return res
