"""Chebyshev-Jacobi p-multigrid preconditioner.

Drop-in for nekmini's ``MultigridHierarchy`` / ``chebyshev_smooth`` /
``pmg_preconditioner`` / ``coarse_solve`` (SPEC.md:466-471, 489-497,
509-527): orders N -> max(N//2, 1) -> 1, a multiplicative
V-cycle with Chebyshev-accelerated Jacobi pre- and post-smoothing on every
level but the coarsest, and an exact coarse solve.

Everything on the V-cycle's path is a libnekb200 launch on the current
stream, on preallocated buffers, so whole PCG iterations are CUDA-graph
captured (MultigridPCG):
  * A at each level: nk_bk5 (+ mask) and the level's gs plan;
  * nk_cheb_step: one fused Chebyshev-Jacobi step (residual update, d, e);
  * nk_interp3: restriction (fused r - A e, 1/mult weight, coarse mask) and
    prolongation (fused mask and accumulate into e);
  * coarse: nk_gather (one copy per unique unmasked dof) -> nk_dense_matvec
    with the explicit inverse of the assembled N = 1 operator -> nk_gather
    back to the L-vector (masked points read a zero slot).
Setup (meshes per order, gs plans, lambda_max by power iteration, the coarse
inverse) runs once on the device through the same library plus torch
linear algebra.

Smoothers (SPEC.md:462-464 SmootherConfig kinds): 'cheby_jac' (default),
'jacobi' (Chebyshev degree 1 = optimally damped Jacobi), 'asm' / 'ras' (one
overlapping-Schwarz FDM application, paper_2104_05829_b200/schwarz.py) and
'cheby_asm' / 'cheby_ras' (Chebyshev acceleration of the Schwarz smoother,
PAPER.md:312-313 CHEBY-ASM).  Schwarz smoothing is not symmetric in the PCG
inner product (the counting weight): use flexible PCG.

Frozen choices (oracle/pmg.py states the same algorithm on the CPU):
degree 2, bounds (0.1, 1.1) x lambda_max of S A for Chebyshev-Jacobi and
(0.4, 1.1) for Chebyshev-Schwarz (SCHWARZ_BOUNDS: with the lower fraction
at SPEC's 0.1 the degree-2 polynomial damps the whole S A spectrum by only
~0.53 and CHEBY-ASM needs MORE iterations than one undamped ASM application,
10 vs 7 on SPEC.md:541's E = 64 problem; 0.4 gives 5 -- measured with the
oracle, profiles/r2_smoother_bounds.jsonl; explicit `bounds` override both),
lambda_max from 20 power iterations from a fixed-seed random start (SPEC's
10 iterations from the ones vector underestimate it by ~30% at N = 7 and make
the smoother amplify the top of the spectrum -- DESIGN.md "p-multigrid").
"""

import numpy as np

from ._lib import ContractError, check, lib, ptr, stream_ptr
from .basis import SpectralBasis, lagrange_interp_matrix
from .gather_scatter import _halo_exchange, _halo_finish, _halo_start, _local
from .mesh import Mesh, assign_global_ids, build_box_mesh, mesh_from_coords

__all__ = ["MultigridHierarchy", "MultigridPCG", "chebyshev_smooth", "pmg_preconditioner",
           "coarse_solve", "chebyshev_coefficients", "pmg_orders", "SMOOTHERS"]

SMOOTHERS = ("jacobi", "cheby_jac", "asm", "ras", "cheby_asm", "cheby_ras")
_SCHWARZ = {"asm": "asm", "ras": "ras", "cheby_asm": "asm", "cheby_ras": "ras"}

# default Chebyshev bound fractions of lambda_max(S A): SPEC.md:548 for the
# Jacobi smoothers, a measured lower fraction for the Schwarz ones (above)
JACOBI_BOUNDS = (0.1, 1.1)
SCHWARZ_BOUNDS = (0.4, 1.1)

DENSE_COARSE_MAX = 16384     # unique unmasked coarse dofs (2 GiB FP64 inverse)


def pmg_orders(N):
    """{N, max(N//2, 1), 1} deduplicated, strictly decreasing."""
    out = []
    for n in (int(N), max(int(N) // 2, 1), 1):
        if n not in out:
            out.append(n)
    return out


def chebyshev_coefficients(degree, lo, hi):
    """Saad's three-term Chebyshev recurrence on [lo, hi] from e0 = 0:
    [(a_0 = 0, b_0 = 1/theta), (a_i, b_i) ...] with d_i = a_i d_{i-1} +
    b_i D^-1 res_i (oracle/pmg.py:chebyshev_smooth)."""
    if degree < 1:
        raise ContractError("Chebyshev degree must be >= 1")
    if not (0.0 < lo < hi):
        raise ContractError(f"invalid eigenvalue bounds ({lo}, {hi})")
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    out = [(0.0, 1.0 / theta)]
    for _ in range(1, degree):
        rho_new = 1.0 / (2.0 * sigma - rho)
        out.append((rho_new * rho, 2.0 * rho_new / delta))
        rho = rho_new
    return out


def _gs(h, w, st=None):
    """In-place QQ^T on the current stream, skipped once st->done."""
    if h.comm is None or h.comm.size == 1:
        _local(h, w, "+", 1, st=st)
        return
    _halo_start(h, w, st=st)
    _halo_exchange(h)
    _local(h, w, "+", 1, st=st, part=h.seg_rest)
    _halo_finish(h, w, "+", st=st)


def _level_mesh(fine, n):
    """The fine mesh's elements at order n: the box map re-evaluated at the
    order-n GLL points, or (explicit-coordinate meshes) the fine coordinates
    interpolated to them, ids re-derived from coordinates and the mask taken
    from the nearest fine node of the same element."""
    if fine.N == n:
        return fine
    if fine.counts is not None:
        return build_box_mesh(fine.extent, fine.counts, n, bc=fine.bc,
                              deformation=fine.deformation, origin=fine.origin,
                              elements=fine.elements, device=fine.device)
    if fine.xyz is None:
        raise ContractError("p-multigrid needs a box mesh or a mesh built with coordinates")
    import torch
    fb, cb = fine.basis, SpectralBasis.get(n)
    M = np.ascontiguousarray(lagrange_interp_matrix(fb.nodes, cb.nodes))   # (n+1, N+1)
    xyz = torch.empty((3, fine.E, n + 1, n + 1, n + 1), dtype=torch.float64, device=fine.device)
    for c in range(3):
        check(lib().nk_interp3(fine.nq, n + 1, fine.E, ptr(M),
                               ptr(fine.xyz[c].contiguous()), None, None, None, ptr(xyz[c]), 0,
                               None, stream_ptr()), "interp3")
    near = np.argmin(np.abs(cb.nodes[:, None] - fb.nodes[None, :]), axis=1)
    fm = fine.mask.reshape(fine.E, fine.nq, fine.nq, fine.nq)
    idx = torch.as_tensor(near, device=fine.device)
    mask = fm[:, idx][:, :, idx][:, :, :, idx].contiguous()
    ids = assign_global_ids(xyz.cpu().numpy())
    return mesh_from_coords(xyz.cpu().numpy(), n, ids=ids, mask=mask.cpu().numpy(),
                            device=fine.device)


class _Level:
    pass


class MultigridHierarchy:
    """p-multigrid hierarchy on a PoissonOperator.

    ``levels[0].op`` is the given operator; coarser levels hold their own
    mesh, PoissonOperator (same lam0, lam1, comm) and Jacobi diagonal.
    Calling the hierarchy applies one V-cycle (pmg_preconditioner).

    coarse: 'dense' (explicit inverse of the assembled, masked order-1
    operator; exact; at most DENSE_COARSE_MAX unique dofs), 'pcg' (fused
    Jacobi-PCG on the order-1 level to coarse_tol relative residual, at most
    coarse_iters iterations -- a nonlinear preconditioner: use flexible PCG),
    or 'auto' (dense when it fits, else pcg).  The paper uses AMG (Hypre /
    parAlmond) here; the iterative coarse solve is the
    scalable stand-in built on the same fused PCG kernels."""

    def __init__(self, op, degree=2, bounds=None, power_iters=20, seed=2104,
                 coarse="auto", smoother="cheby_jac", smoother_precision=64, coarse_tol=1e-2,
                 coarse_iters=50):
        import torch
        from .solvers import JacobiPreconditioner, PoissonOperator
        if op.ncomp != 1:
            raise ContractError("p-multigrid preconditions scalar operators")
        if coarse not in ("dense", "pcg", "auto"):
            raise ContractError(f"unknown coarse solver {coarse!r} (built: 'dense', 'pcg', "
                                f"'auto')")
        self.coarse_kind = coarse
        self.coarse_tol, self.coarse_iters = float(coarse_tol), int(coarse_iters)
        self.comm = op.comm if (op.comm is not None and op.comm.size > 1) else None
        if self.comm is not None:
            # across ranks: box meshes (each rank rebuilds its own elements at
            # every order), any smoother (the Schwarz boxes read the neighbour
            # ranks' face layers from one exchange per smoothing; ASM's
            # extended gs runs over the ranks) and the iterative coarse solve
            # (the fused PCG runs over the same halo + all-reduce path)
            if op.mesh.counts is None:
                raise ContractError("multi-rank p-multigrid needs a box mesh")

            if coarse == "dense":
                raise ContractError("the dense coarse solve is single-rank: use coarse='pcg'")
        if bounds is None:
            bounds = SCHWARZ_BOUNDS if smoother in ("cheby_asm", "cheby_ras") else JACOBI_BOUNDS
        if not (0.0 < bounds[0] < bounds[1]):
            raise ContractError(f"invalid eigenvalue bound fractions {bounds}")
        self.degree = int(degree)
        if self.degree < 1:
            raise ContractError("Chebyshev degree must be >= 1")
        if smoother not in SMOOTHERS:
            raise ContractError(f"unknown smoother {smoother!r} (built: {SMOOTHERS})")
        self.smoother = smoother
        if smoother_precision not in (32, 64):
            raise ContractError(f"smoother_precision must be 32 or 64, got {smoother_precision!r}")
        if smoother_precision == 32 and smoother not in _SCHWARZ:
            raise ContractError("32-bit smoothing is built for the Schwarz (FDM) smoothers")
        self.smoother_precision = int(smoother_precision)
        self.bounds = (float(bounds[0]), float(bounds[1]))
        self.orders = pmg_orders(op.mesh.N)
        dev = op.mesh.device
        self.levels = []
        for n in self.orders:
            lv = _Level()
            lv.order, lv.nq = n, n + 1
            if n == op.mesh.N:
                lv.mesh, lv.op = op.mesh, op
            else:
                lv.mesh = _level_mesh(op.mesh, n)
                lv.op = PoissonOperator(lv.mesh, lam0=op.lam0, lam1=op.lam1, comm=op.comm)
            lv.n = lv.mesh.n_local
            lv.invD = JacobiPreconditioner(lv.op).invD
            lv.wt = lv.op.weights
            lv.mask = lv.mesh.mask.reshape(-1)
            f = lambda: torch.zeros(lv.n, dtype=torch.float64, device=dev)
            lv.e, lv.d, lv.res, lv.Aq = f(), f(), f(), f()
            lv.r = f() if self.levels else None
            lv.kind = smoother
            lv.sm = None
            lv.gate_partials = torch.zeros(lv.op.partials_len(), dtype=torch.float64, device=dev)
            self.levels.append(lv)
        from .schwarz import SchwarzSmoother
        for lv in self.levels[:-1]:
            if smoother in _SCHWARZ:
                lv.sm = SchwarzSmoother(lv.op, _SCHWARZ[smoother], precision=smoother_precision)
                lv.res2 = torch.zeros_like(lv.res)
            lv.deg = 1 if smoother in ("jacobi", "asm", "ras") else self.degree
        for lv in self.levels[:-1]:
            lv.lmax = self._power_lambda_max(lv, power_iters, seed)
            if not lv.lmax > 0.0:
                raise ContractError(f"lambda_max estimate {lv.lmax} <= 0 (order {lv.order})")
            lv.lo, lv.hi = self.bounds[0] * lv.lmax, self.bounds[1] * lv.lmax
            lv.coef = chebyshev_coefficients(lv.deg, lv.lo, lv.hi)
        for f, c in zip(self.levels[:-1], self.levels[1:]):
            J = lagrange_interp_matrix(c.mesh.basis.nodes, f.mesh.basis.nodes)  # (nq_f, nq_c)
            f.P = np.ascontiguousarray(J)
            f.R = np.ascontiguousarray(J.T)
        self._coarse_setup(self.levels[-1])

    # ---------------------------------------------------------------- setup
    def _power_lambda_max(self, lv, iters, seed):
        """lambda_max of D^-1 A: power iteration with the 1/mult-weighted norm
        from mask * QQ^T (wt * random(seed)) (oracle/pmg.py:power_lambda_max)."""
        import torch
        x0 = np.random.default_rng(seed).standard_normal(lv.n)
        x = torch.as_tensor(x0, device=lv.mesh.device) * lv.wt
        _gs(lv.op.gs, x)
        x = x * lv.mask.to(x.dtype)
        y = torch.empty_like(x)
        lam = 0.0
        nrm = torch.zeros(2, dtype=torch.float64, device=x.device)
        for _ in range(int(iters)):
            lv.op.apply(x, y)
            if lv.sm is not None:
                y = lv.sm(y)
            else:
                y = lv.invD * y
            nrm[0] = torch.sum(lv.wt * y * y)
            nrm[1] = torch.sum(lv.wt * x * x)
            if self.comm is not None:
                self.comm.allreduce_sum_(nrm)
            ny, nx = (float(v) for v in torch.sqrt(nrm).cpu())
            lam = ny / nx
            x = y / ny
            y = torch.empty_like(x)
        return lam

    def _coarse_setup(self, lv):
        """Explicit inverse of the assembled, masked coarse operator on the
        unique unmasked dofs.  Element matrices come from
        nq^3 BK5 launches on unit vectors (column k of every element at
        once); assembly and the Cholesky inverse run once on the device.
        Pure Neumann/periodic with lam1 = 0: the constant is projected out,
        Ainv = (A + 1 1^T)^-1 - 1 1^T / n^2."""
        import torch
        from .kernels import _bk5
        if self.comm is not None:
            lv.nu = -1                 # distributed: no global unique numbering here
            self._coarse_setup_pcg(lv)
            return
        m, dev = lv.mesh, lv.mesh.device
        nq3 = lv.nq ** 3
        ids = m.ids.reshape(-1)
        mask = lv.mask.bool()
        uniq, inv = torch.unique(ids, return_inverse=True)
        # a unique id is kept when unmasked (the mask agrees on every copy)
        keep_u = torch.zeros(uniq.numel(), dtype=torch.bool, device=dev)
        keep_u[inv[mask]] = True
        nu = int(keep_u.sum())
        lv.nu = nu
        if self.coarse_kind == "pcg" or (self.coarse_kind == "auto" and nu > DENSE_COARSE_MAX):
            self._coarse_setup_pcg(lv)
            return
        if nu > DENSE_COARSE_MAX:
            raise ContractError(f"coarse problem has {nu} unique dofs > {DENSE_COARSE_MAX}: "
                                f"use coarse='pcg' (or 'auto')")
        lv.cpcg = None
        newid = torch.full((uniq.numel(),), -1, dtype=torch.int64, device=dev)
        newid[keep_u] = torch.arange(nu, device=dev)
        uid = newid[inv]                                  # per local point, -1 masked
        u = torch.zeros((m.E, nq3), dtype=torch.float64, device=dev)
        cols = []
        for k in range(nq3):
            u.zero_()
            u[:, k] = 1.0
            cols.append(_bk5(u.reshape(-1), m, lv.op.lam0, lv.op.lam1, 1).reshape(m.E, nq3))
        Ae = torch.stack(cols, dim=2)                     # Ae[e, a, k]
        ul = uid.reshape(m.E, nq3)
        rows = ul[:, :, None].expand(m.E, nq3, nq3)
        colsi = ul[:, None, :].expand(m.E, nq3, nq3)
        ok = (rows >= 0) & (colsi >= 0)
        A = torch.zeros((nu, nu), dtype=torch.float64, device=dev)
        A.index_put_((rows[ok], colsi[ok]), Ae[ok], accumulate=True)
        A = 0.5 * (A + A.T)
        singular = (not bool(mask.logical_not().any())) and lv.op.lam1 == 0.0
        if singular:
            A = A + 1.0
        Lc, info = torch.linalg.cholesky_ex(A)
        if int(info) != 0:
            raise ContractError("coarse factorization failed: the assembled order-1 operator "
                                "is not positive definite")
        Ainv = torch.cholesky_inverse(Lc)
        if singular:
            Ainv = Ainv - 1.0 / float(nu) ** 2
        lv.Ainv = Ainv.contiguous()
        # 32-bit smoothing mode: the coarse inverse streams as FP32 (half the
        # bytes of the one n^2 pass per V-cycle; sums stay FP64)
        lv.Ainv32, lv.lda = None, (nu + 3) // 4 * 4
        if self.smoother_precision == 32:
            lv.Ainv32 = torch.zeros((nu, lv.lda), dtype=torch.float32, device=dev)
            lv.Ainv32[:, :nu] = Ainv.float()
        lv.nu = nu
        # representative local copy of each kept unique id, and the scatter map
        # (masked points -> slot nu, which stays zero)
        rep = torch.full((nu,), -1, dtype=torch.int64, device=dev)
        kept = uid >= 0
        pos = torch.arange(uid.numel(), device=dev)
        rep.scatter_reduce_(0, uid[kept], pos[kept], reduce="amin", include_self=False)
        lv.rep = rep.to(torch.int32)
        lv.scat = torch.where(kept, uid, torch.full_like(uid, nu)).to(torch.int32)
        lv.ru = torch.zeros((nu + 3) // 4 * 4, dtype=torch.float64, device=dev)   # lda-padded
        lv.eu = torch.zeros(nu + 1, dtype=torch.float64, device=dev)

    # ---------------------------------------------------------------- apply
    def _apply_A(self, lv, x, y, st=None):
        """y = A x on a level; with the PCG state, the launches are skipped
        once the outer solve is done (graph replays past convergence)."""
        if st is None or lv.op.gs.comm is not None and lv.op.gs.comm.size > 1:
            lv.op.apply(x, y)
        else:
            lv.op.apply(x, y, st=st, partials=lv.gate_partials, reduce=False)

    def _cheb(self, lv, r, st, post):
        """Smoothing of A e = r into lv.e.  Pre: e = S r.  Post (r = the
        level's right-hand side, lv.Aq = A e on entry): e += S (r - A e).
        (oracle/pmg.py:smooth / chebyshev_smooth)"""
        if lv.sm is not None:
            self._cheb_schwarz(lv, r, st, post)
            return
        L, s = lib(), stream_ptr()
        deg = lv.deg
        a0, b0 = lv.coef[0]
        keep_res = deg > 1
        check(L.nk_cheb_step(lv.n, ptr(r), ptr(lv.Aq) if post else None, ptr(lv.invD),
                             ptr(lv.res) if (post and keep_res) else None, ptr(lv.d), ptr(lv.e),
                             a0, b0, int(post), ptr(st), s), "cheb_step")
        src = lv.res if post else r
        for i in range(1, deg):
            self._apply_A(lv, lv.d, lv.Aq, st)
            a, b = lv.coef[i]
            store = lv.res if i < deg - 1 else None
            check(L.nk_cheb_step(lv.n, ptr(src), ptr(lv.Aq), ptr(lv.invD), ptr(store),
                                 ptr(lv.d), ptr(lv.e), a, b, 1, ptr(st), s), "cheb_step")
            src = lv.res

    def _cheb_schwarz(self, lv, r, st, post):
        """Schwarz smoothing: 'asm'/'ras' one application; cheby_* the
        Chebyshev recurrence with the Schwarz solve as inner smoother.  The
        residual update r - A d is fused into the FDM gather (sub = A d);
        residuals ping-pong between two buffers (the gather reads neighbour
        points of the buffer the previous step wrote)."""
        sm = lv.sm
        if lv.kind in ("asm", "ras"):
            sm.apply(r, lv.e, sub=lv.Aq if post else None, e_acc=post, st=st)
            return
        deg = lv.deg
        bufs = (lv.res, lv.res2)
        a0, b0 = lv.coef[0]
        store = bufs[0] if (post and deg > 1) else None
        sm.apply(r, lv.e, sub=lv.Aq if post else None, res_out=store, d=lv.d, a=a0, b=b0,
                 e_acc=post, st=st)
        src = store if post else r
        for i in range(1, deg):
            self._apply_A(lv, lv.d, lv.Aq, st)
            a, b = lv.coef[i]
            store = bufs[i % 2] if i < deg - 1 else None
            sm.apply(src, lv.e, sub=lv.Aq, res_out=store, d=lv.d, a=a, b=b, e_acc=True, st=st)
            src = store

    def _coarse_setup_pcg(self, lv):
        from .solvers import FusedPCG, JacobiPreconditioner
        # one kernel per fused step here: the coarse levels are small and
        # launch-bound, where a 4th launch per iteration costs more than the
        # split saves (the split_step default is measured at ~3M points)
        lv.cpcg = FusedPCG(lv.op, JacobiPreconditioner(lv.op), tol=self.coarse_tol,
                           max_iter=self.coarse_iters, use_graph=False, split_step=False)
        lv.e = lv.cpcg.x           # the coarse correction is the inner solution

    def _coarse(self, lv, r, st):
        L, s = lib(), stream_ptr()
        if lv.cpcg is not None:
            # fixed launch sequence (graph-capturable): init + max_iter + 1
            # fused iterations; converged iterations are no-ops, the last one
            # applies the deferred x update
            c = lv.cpcg
            c.init(r)
            if st is not None:       # no-op once the outer PCG is done
                check(L.nk_cg_gate(ptr(c.st), ptr(st), s), "cg_gate")
            for _ in range(self.coarse_iters + 1):
                c._iteration()
            return
        check(L.nk_gather(lv.nu, ptr(lv.rep), ptr(r), ptr(lv.ru), ptr(st), s), "gather")
        if getattr(lv, "Ainv32", None) is not None:
            check(L.nk_dense_matvec32(lv.nu, lv.lda, ptr(lv.Ainv32), ptr(lv.ru), ptr(lv.eu),
                                      ptr(st), s), "dense_matvec32")
        else:
            check(L.nk_dense_matvec(lv.nu, ptr(lv.Ainv), ptr(lv.ru), ptr(lv.eu), ptr(st), s),
                  "dense_matvec")
        check(L.nk_gather(lv.n, ptr(lv.scat), ptr(lv.eu), ptr(lv.e), ptr(st), s), "gather")

    def _vcycle(self, k, r, st):
        L, s = lib(), stream_ptr()
        lv = self.levels[k]
        if k == len(self.levels) - 1:
            self._coarse(lv, r, st)
            return
        c = self.levels[k + 1]
        self._cheb(lv, r, st, post=False)                         # pre-smooth
        self._apply_A(lv, lv.e, lv.Aq, st)
        check(L.nk_interp3(lv.nq, c.nq, lv.mesh.E, ptr(lv.R), ptr(r), ptr(lv.Aq), ptr(lv.wt),
                           ptr(c.mask), ptr(c.r), 0, ptr(st), s), "interp3")   # restrict
        _gs(c.op.gs, c.r, st)
        self._vcycle(k + 1, c.r, st)
        check(L.nk_interp3(c.nq, lv.nq, lv.mesh.E, ptr(lv.P), ptr(c.e), None, None,
                           ptr(lv.mask), ptr(lv.e), 1, ptr(st), s), "interp3")  # prolong
        self._apply_A(lv, lv.e, lv.Aq, st)
        self._cheb(lv, r, st, post=True)                          # post-smooth

    def apply(self, r, st=None):
        """z = M^-1 r (one V-cycle); returns the level-0 buffer holding z
        (overwritten by the next call)."""
        lv = self.levels[0]
        if r.numel() != lv.n:
            raise ContractError(f"contract error: field length {r.numel()} != {lv.n}")
        self._vcycle(0, r.reshape(-1), st)
        return lv.e

    def __call__(self, r):
        return self.apply(r).view_as(r)

    @property
    def launches_per_vcycle(self):
        """Library launches in one V-cycle (for bench gpu_launches)."""
        import torch  # noqa: F401
        n = 0
        for lv in self.levels[:-1]:
            g = 1                                             # gs (single rank)
            A = 1 + g
            per = 3 if lv.sm is not None else 1               # fdm + gs + post | cheb step
            n += 2 * lv.deg * per                             # smoothing steps (pre + post)
            n += 2 * (lv.deg - 1) * A                         # A d inside smoothing
            n += 2 * A                                        # A e before restrict / after prolong
            n += 2 + g                                        # interp x2, coarse gs
        c = self.levels[-1]
        if getattr(c, "cpcg", None) is not None:
            return n + 3 + 3 * (self.coarse_iters + 1)
        return n + 3


def chebyshev_smooth(hierarchy, level, r, degree=None):
    """Correction e = S r of one smoothing (e0 = 0) with the hierarchy's
    smoother at `level` (degree overrides the Chebyshev
    degree).  Returns a new tensor."""
    h = hierarchy
    lv = h.levels[level]
    if level == len(h.levels) - 1:
        raise ContractError("the coarsest level is solved directly, not smoothed")
    old = lv.deg, lv.coef
    if degree is not None and int(degree) != lv.deg:
        if int(degree) < 1:
            raise ContractError("Chebyshev degree must be >= 1")
        lv.deg = int(degree)
        lv.coef = chebyshev_coefficients(lv.deg, lv.lo, lv.hi)
    try:
        h._cheb(lv, r.reshape(-1).contiguous(), None, post=False)
    finally:
        lv.deg, lv.coef = old
    return lv.e.clone().view_as(r)


def pmg_preconditioner(hierarchy, r):
    """z = one V-cycle applied to r; a new tensor."""
    return hierarchy.apply(r.reshape(-1).contiguous()).clone().view_as(r)


def coarse_solve(hierarchy, rhs):
    """Exact solve with the assembled order-1 operator:
    rhs is an assembled, masked L-vector at order 1; returns the L-vector."""
    lv = hierarchy.levels[-1]
    r = rhs.reshape(-1).contiguous()
    if r.numel() != lv.n:
        raise ContractError(f"contract error: field length {r.numel()} != {lv.n}")
    hierarchy._coarse(lv, r, None)
    return lv.e.clone().view_as(rhs)


class MultigridPCG:
    """Graph-captured PCG preconditioned by one p-multigrid V-cycle.

    Per iteration: nk_bk5 (w = A p, p^T A p fused) + gs, nk_cg_update
    (x, r, <r, r>_w), the V-cycle (z = M^-1 r), nk_wdot (<r, z>_w [, <z, Ap>_w
    for flexible]), nk_cg_pupdate (beta, p, test).  ``chunk`` iterations per
    graph replay; once the device flag is set, every launch is a no-op except
    the V-cycle's BK5s (they carry no state pointer)."""

    def __init__(self, op, hierarchy=None, tol=1e-8, max_iter=500, flexible=None, chunk=4,
                 use_graph=True, **hier_kw):
        import torch
        from .solvers import _state_tensor
        self.op = op
        self.h = hierarchy if hierarchy is not None else MultigridHierarchy(op, **hier_kw)
        if flexible is None:
            # non-symmetric (Schwarz counting weight) or nonlinear (iterative
            # coarse solve) preconditioners need the flexible beta
            flexible = (self.h.smoother in _SCHWARZ or
                        getattr(self.h.levels[-1], "cpcg", None) is not None)
        self.tol, self.max_iter, self.flexible = float(tol), int(max_iter), bool(flexible)
        self.chunk = max(1, int(chunk))
        self.use_graph = use_graph
        dev = op.mesh.device
        n = self.n = op.n
        f = lambda: torch.zeros(n, dtype=torch.float64, device=dev)
        self.x, self.r, self.p, self.w = f(), f(), f(), f()
        self.st = _state_tensor(dev)
        self.s64 = self.st.view(torch.float64)
        self.part_bk5 = torch.zeros(op.partials_len(), dtype=torch.float64, device=dev)
        self.part_cg = torch.zeros(int(lib().nk_cg_partials_len(n)), dtype=torch.float64,
                                   device=dev)
        self.part_dot = torch.zeros_like(self.part_cg)
        self.hist = torch.zeros(self.max_iter + 2, dtype=torch.float64, device=dev)
        self.wt = op.weights
        self.graph = None
        comm = op.gs.comm
        self.comm = comm if (comm is not None and comm.size > 1) else None
        if self.comm is not None:
            board = False
            if getattr(op.gs, "transport", "p2p") == "ipc":
                board = self.comm.enable_board(dev)
            # graph capture needs every exchange on the stream; the Schwarz
            # face-layer exchange goes through torch.distributed
            schwarz = any(lv.sm is not None for lv in self.h.levels)
            self.use_graph = self.use_graph and (
                self.comm.staging == "device" or (board and not schwarz))

    def _allreduce(self, a, b):
        if self.comm is not None:
            self.comm.allreduce_sum_(self.s64[a:b])

    @property
    def launches_per_iter(self):
        return 2 + 1 + self.h.launches_per_vcycle + 2 * (2 if self.flexible else 1) + 1

    def _iteration(self):
        L, s = lib(), stream_ptr()
        n = self.n
        self.op.apply(self.p, self.w, st=self.st, partials=self.part_bk5)      # pAp
        self._allreduce(1, 2)
        check(L.nk_cg_update(n, ptr(self.x), ptr(self.r), ptr(self.p), ptr(self.w), None,
                             ptr(self.wt), None, ptr(self.st), ptr(self.part_cg), s),
              "cg_update")
        self._allreduce(3, 4)                                                  # rr
        z = self.h.apply(self.r, self.st)
        check(L.nk_wdot(n, ptr(self.r), ptr(z), ptr(self.wt), ptr(self.s64[2:3]),
                        ptr(self.part_dot), s), "wdot")
        self._allreduce(2, 3)                                                  # rz_new
        if self.flexible:
            check(L.nk_wdot(n, ptr(z), ptr(self.w), ptr(self.wt), ptr(self.s64[4:5]),
                            ptr(self.part_dot), s), "wdot")
            self._allreduce(4, 5)                                              # zAp
        check(L.nk_cg_pupdate(n, ptr(self.r), ptr(self.p), None, ptr(z), ptr(self.st),
                              ptr(self.hist), s), "cg_pupdate")

    def init(self, b):
        L, s = lib(), stream_ptr()
        n = self.n
        bf = b.reshape(-1)
        if bf.numel() != n:
            raise ContractError(f"contract error: field length {bf.numel()} != {n}")
        self.b = bf.contiguous()
        self.st.zero_()
        check(L.nk_cg_init(n, ptr(self.b), ptr(self.x), ptr(self.r), ptr(self.p), None,
                           ptr(self.wt), ptr(self.st), ptr(self.part_cg), self.tol,
                           self.max_iter, int(self.flexible), s), "cg_init")
        check(L.nk_wdot(n, ptr(self.b), ptr(self.b), ptr(self.wt), ptr(self.s64[5:6]),
                        ptr(self.part_dot), s), "wdot")
        self._allreduce(3, 4)                                                  # rr
        self._allreduce(5, 6)                                                  # bb
        z = self.h.apply(self.r)
        self.p.copy_(z)
        check(L.nk_wdot(n, ptr(self.r), ptr(z), ptr(self.wt), ptr(self.s64[0:1]),
                        ptr(self.part_dot), s), "wdot")
        self._allreduce(0, 1)                                                  # rz
        check(L.nk_cg_init_finalize(ptr(self.st), ptr(self.hist), s), "cg_init_finalize")

    def _capture(self):
        import torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(self.chunk):
                self._iteration()
        return g

    def run(self):
        import torch
        from .solvers import read_state
        from .kernels import COUNTERS
        if self.use_graph and self.graph is None:
            # warm-up outside capture (first-call attribute setup), then reset;
            # KernelCounters: the warm-up and the re-init are not counted, one
            # captured chunk is recorded and added per executed iteration
            with COUNTERS.recording():
                self._iteration()
                torch.cuda.synchronize()
            with COUNTERS.recording() as rec:
                self.graph = self._capture()
            self._iter_counts = (rec, self.chunk)
            with COUNTERS.recording():
                self.init(self.b)
        stt = read_state(self.st)
        while not stt.done:
            if self.use_graph:
                self.graph.replay()
            else:
                with COUNTERS.recording() as rec:
                    for _ in range(self.chunk):
                        self._iteration()
                self._iter_counts = (rec, self.chunk)
            stt = read_state(self.st)
        return stt

    def solve(self, b):
        from .solvers import BreakdownError, PCGResult
        self.init(b)
        stt = self.run()
        if stt.breakdown:
            raise BreakdownError(f"p^T A p <= 0 at iteration {stt.iter}")
        it = int(stt.iter)
        from .solvers import _count_iterations
        _count_iterations(self, it)
        hist = self.hist[:it + 1].cpu().numpy().tolist()
        return PCGResult(self.x.view_as(b), it, hist, bool(stt.converged))
