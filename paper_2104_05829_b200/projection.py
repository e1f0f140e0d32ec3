"""Projection-based initial guesses.

Drop-in for nekmini's ``ProjectionSpace`` / ``project_guess`` / ``update``
(SPEC.md:472-475 type, 529-537 operations): successive
solves with slowly varying right-hand sides (pressure at consecutive time
steps) start from the A-projection of b onto the span of the last
``capacity`` solutions.

Device-resident: the stored A-orthonormal basis X (capacity rows; the
oldest is evicted before the candidate is orthonormalised, so x_new always
lies in the span afterwards) and A X live in HBM, coefficients live
in device memory, and every pass is a libnekb200 launch
(nk_multi_wdot, nk_multi_axpy, nk_vscale) on the current stream:
  project  1 multi-dot over b + 2 multi-axpy      ((k + 2) + 2 (k + 2) vectors)
  update   2 x (multi-dot + 2 multi-axpy) (CGS2), 1 dot, 2 scalings
The only host synchronisation is the degeneracy test of ``update`` (once per
solve).  Inner products are over unique dofs (1/mult-weighted L-vector dots,
the PCG convention of SPEC.md:482), reduced in fixed order and all-reduced
over ranks when the operator is distributed.

The algorithm is restated on the CPU in oracle/projection.py.
"""

from ._lib import ContractError, check, lib, ptr, stream_ptr

__all__ = ["ProjectionSpace", "project_guess", "update", "ProjectedSolver"]

DEGENERATE = 1e-10


class ProjectionSpace:
    """Up to ``capacity`` A-orthonormal prior solutions of ``op`` (a
    PoissonOperator); x_i^T A x_j = delta_ij."""

    def __init__(self, op, capacity=8):
        import torch
        capacity = int(capacity)
        if op.ncomp != 1:
            raise ContractError("projection spaces hold scalar fields (one space per component)")
        if not 1 <= capacity < 16:
            raise ContractError(f"projection capacity must be in [1, 15], got {capacity}")
        self.op, self.capacity = op, capacity
        dev = op.mesh.device
        n = self.n = op.n
        f = lambda *s: torch.zeros(*s, dtype=torch.float64, device=dev)
        self.X = f(capacity, n)
        self.AX = f(capacity, n)
        self.c = f(16)
        self.s = f(4)
        self.partials = f(int(lib().nk_multi_wdot_partials_len()))
        self.wt = op.weights
        self.k = 0
        self.restarts = 0
        comm = op.gs.comm if op.gs is not None else None
        self.comm = comm if (comm is not None and comm.size > 1) else None

    @property
    def size(self):
        return self.k

    def clear(self):
        self.k = 0

    # ------------------------------------------------------------ primitives
    def _mdot(self, k, y, out):
        """out[:k] = <X[q], y>_w for q < k (all-reduced)."""
        check(lib().nk_multi_wdot(self.n, k, ptr(self.X), self.n, ptr(y), ptr(self.wt), ptr(out),
                                  ptr(self.partials), stream_ptr()), "multi_wdot")
        if self.comm is not None:
            self.comm.allreduce_sum_(out[:k])

    def _dot(self, a, b, out):
        check(lib().nk_multi_wdot(self.n, 1, ptr(a), self.n, ptr(b), ptr(self.wt), ptr(out),
                                  ptr(self.partials), stream_ptr()), "multi_wdot")
        if self.comm is not None:
            self.comm.allreduce_sum_(out[:1])

    def _axpy(self, k, scale, V, yin, yout):
        check(lib().nk_multi_axpy(self.n, k, ptr(self.c), scale, ptr(V), self.n, ptr(yin),
                                  ptr(yout), stream_ptr()), "multi_axpy")

    def _check(self, t):
        import torch
        if (not isinstance(t, torch.Tensor) or t.numel() != self.n or t.dtype != torch.float64
                or not t.is_cuda):
            raise ContractError(f"contract error: field must be a CUDA float64 tensor of "
                                f"{self.n} values")
        return t.reshape(-1).contiguous()

    # ------------------------------------------------------------ operations
    def project(self, b, x0=None, bdef=None):
        """x0 = sum_i <x_i, b> x_i and b' = b - sum_i <x_i, b> A x_i
        (SPEC.md:529-532).  Returns (x0, b'), new tensors unless given."""
        import torch
        bf = self._check(b)
        x0 = torch.empty_like(bf) if x0 is None else x0.reshape(-1)
        bdef = torch.empty_like(bf) if bdef is None else bdef.reshape(-1)
        k = self.k
        if k == 0:
            x0.zero_()
            bdef.copy_(bf)
            return x0.view_as(b), bdef.view_as(b)
        self._mdot(k, bf, self.c)
        self._axpy(k, 1.0, self.X, None, x0)
        self._axpy(k, -1.0, self.AX, bf, bdef)
        return x0.view_as(b), bdef.view_as(b)

    def update(self, x_new, Ax_new=None):
        """Append the A-orthonormalised x_new: evict the
        oldest when full, CGS2 against the rest, restart (keep only
        x_new) when ||candidate||_A < 1e-10 ||x_new||_A.  Ax_new (= A x_new,
        assembled) is computed with the operator when not given."""
        xf = self._check(x_new)
        if self.k >= self.capacity:                         # evict the oldest first
            k = self.k
            self.X[:k - 1].copy_(self.X[1:k].clone())
            self.AX[:k - 1].copy_(self.AX[1:k].clone())
            self.k = k - 1
        cand, acand = self.X[self.k], self.AX[self.k]
        cand.copy_(xf)
        if Ax_new is None:
            self.op.apply(cand, acand)
        else:
            acand.copy_(self._check(Ax_new))
        self._dot(cand, acand, self.s[0:1])                 # ||x_new||_A^2
        for _ in range(2 if self.k else 0):                 # CGS2
            self._mdot(self.k, acand, self.c)
            self._axpy(self.k, -1.0, self.X, cand, cand)
            self._axpy(self.k, -1.0, self.AX, acand, acand)
        self._dot(cand, acand, self.s[1:2])                 # ||candidate||_A^2
        n0, n2 = (float(v) for v in self.s[:2].cpu())
        if not n0 > 0.0:
            return
        if not n2 > DEGENERATE ** 2 * n0:
            # restart: the space keeps only x_new
            self.restarts += 1
            self.k = 0
            cand, acand = self.X[0], self.AX[0]
            cand.copy_(xf)
            if Ax_new is None:
                self.op.apply(cand, acand)
            else:
                acand.copy_(self._check(Ax_new))
            self.s[1:2].copy_(self.s[0:1])
        L, st = lib(), stream_ptr()
        check(L.nk_vscale(self.n, ptr(cand), ptr(cand), ptr(self.s[1:2]), st), "vscale")
        check(L.nk_vscale(self.n, ptr(acand), ptr(acand), ptr(self.s[1:2]), st), "vscale")
        self.k += 1

    def gram(self):
        """X^T A X over the stored basis (k x k host array; test helper)."""
        import numpy as np
        import torch
        k = self.k
        G = np.zeros((k, k))
        out = torch.zeros(16, dtype=torch.float64, device=self.X.device)
        for j in range(k):
            self._mdot(k, self.AX[j], out)
            G[:, j] = out[:k].cpu().numpy()
        return G


def project_guess(space, b, apply_A=None):
    """(x0, deflated rhs) -- SPEC.md:529.  apply_A is accepted for API parity;
    the space stores A x_i, so no operator application is needed."""
    return space.project(b)


def update(space, x_new, apply_A=None):
    """SPEC.md:529 update(space, x_new)."""
    Ax = None
    if apply_A is not None and apply_A is not space.op:
        Ax = apply_A(x_new)
    space.update(x_new, Ax)


class ProjectedSolver:
    """A solver (FusedPCG / MultigridPCG / anything with ``tol`` and
    ``solve(b)``) wrapped with a projection space: x0, b' = project(b); solve
    A dx = b' to tol * ||b|| (0 iterations if ||b'|| <= tol ||b||); x = x0 +
    dx; update(x).  Returns the inner solver's PCGResult with x replaced."""

    def __init__(self, solver, space=None, capacity=8):
        self.solver = solver
        self.space = space if space is not None else ProjectionSpace(solver.op, capacity)
        self.tol = float(solver.tol)

    def solve(self, b):
        import math

        import torch
        from .solvers import PCGResult
        sp = self.space
        bf = sp._check(b)
        x0, bd = sp.project(bf)
        out = torch.zeros(2, dtype=torch.float64, device=bf.device)
        sp._dot(bf, bf, out[0:1])
        sp._dot(bd, bd, out[1:2])
        nb2, nd2 = (float(v) for v in out.cpu())
        nb, nd = math.sqrt(max(nb2, 0.0)), math.sqrt(max(nd2, 0.0))
        if nb == 0.0 or nd <= self.tol * nb:
            res = PCGResult(x0.clone().view_as(b), 0, [nd], True)
        else:
            self.solver.tol = self.tol * nb / nd
            try:
                r = self.solver.solve(bd.view_as(b))
            finally:
                self.solver.tol = self.tol
            x = (x0 + r.x.reshape(-1)).view_as(b)
            res = r._replace(x=x)
        sp.update(res.x)
        return res
