"""Preconditioned CG -- the drop-in for ``nekmini.solvers.pcg``
plus the fused B200 Poisson/Helmholtz solve (BP5) built on it.

Two paths, identical iteration structure (Ap, alpha, x/r update, ||r|| test,
z = M r, beta, p update -- SURVEY.md §3 call stack 4):

* ``pcg(apply_A, apply_M, b, ...)`` with arbitrary callables: vector work
  and dots run in the fused CG kernels (nk_cg_update / nk_cg_pupdate /
  nk_wdot); scalars stay on the device; one host sync per iteration for the
  convergence test.
* ``pcg(op, jac, b, ...)`` with ``op`` a :class:`PoissonOperator` and ``jac``
  its :class:`JacobiPreconditioner` takes the fused path (``FusedPCG``): the
  BK5 launch also produces p^T A p, the Jacobi z = invD r is folded into the
  update kernels, and ``chunk`` iterations are captured in one CUDA graph that
  is replayed until the device-side ``done`` flag is set (kernels no-op after
  convergence), so the host syncs once per chunk instead of per iteration.

Dots are weighted by 1/multiplicity, so <a,b>_w is the assembled l2 product
and ||r||_w is the plain 2-norm of the assembled residual.
"""

import ctypes
from collections import namedtuple

import numpy as np

from ._lib import CG_STATE_BYTES, CGState, ContractError, check, lib, ptr, stream_ptr
from .gather_scatter import _halo_exchange, _halo_finish, _halo_start, _local, gs_op, gs_setup
from .kernels import COUNTERS, bk5_flops, extract_diagonal

__all__ = ["pcg", "PCGResult", "BreakdownError", "PoissonOperator", "JacobiPreconditioner",
           "FusedPCG", "FusedPCG3", "inverse_multiplicity", "HelmholtzVectorSolver"]

PCGResult = namedtuple("PCGResult", "x iterations residual_history converged")


class BreakdownError(RuntimeError):
    """p^T A p <= 0."""


def _aligned16(*ts):
    return all(t is None or t.data_ptr() % 16 == 0 for t in ts)


def _state_tensor(device):
    import torch
    return torch.zeros(CG_STATE_BYTES, dtype=torch.uint8, device=device)


def read_state(st):
    raw = st.cpu().numpy().tobytes()
    return CGState.from_buffer_copy(raw)


def inverse_multiplicity(handle, n, device):
    """1/mult per local point via gs(+) on ones (the l2 dot weight)."""
    import torch
    one = torch.ones(n, dtype=torch.float64, device=device)
    gs_op(handle, one)
    return 1.0 / one


class PoissonOperator:
    """A = mask * QQ^T (lam0 A_L + lam1 B) on one rank's L-vectors -- the
    `apply_A` the SPEC's pressure/viscous steps hand to pcg.

    gs may be a handle from gs_setup(mesh.ids, comm, nq=mesh.nq) for multi-rank
    meshes; with comm set the halo exchange overlaps the interior-element BK5
    (boundary elements first)."""

    def __init__(self, mesh, gs=None, lam0=1.0, lam1=0.0, comm=None, ncomp=1):
        self.mesh = mesh
        self.lam0, self.lam1 = float(lam0), float(lam1)
        self.ncomp = ncomp
        self.comm = comm
        self.gs = gs if gs is not None else gs_setup(mesh.ids, comm=comm, nq=mesh.nq,
                                                     device=mesh.device)
        self.n = mesh.n_local
        self._wt = None
        self._mult = None

    @property
    def weights(self):
        if self._wt is None:
            self._wt = inverse_multiplicity(self.gs, self.n, self.mesh.device)
        return self._wt

    @property
    def multiplicity_u8(self):
        """Global multiplicity of every local point as uint8 (the fused CG
        update reads 1 byte instead of an FP64 weight)."""
        import torch
        if self._mult is None:
            one = torch.ones(self.n, dtype=torch.float64, device=self.mesh.device)
            gs_op(self.gs, one)
            if float(one.max()) > 255:
                raise ContractError("multiplicity > 255 cannot be stored as uint8")
            self._mult = torch.round(one).to(torch.uint8)
        return self._mult

    def __call__(self, p, out=None):
        import torch
        if out is None:
            out = torch.empty_like(p)
        self.apply(p, out)
        return out

    def apply(self, p, w, st=None, partials=None, reduce=True, local=None):
        """w = A p (masked, assembled).  With st/partials the BK5 launch also
        stores p^T A p (the rank-local part) in st->pAp; with reduce=False the
        state only gates the launches (no-ops once st->done, e.g. inside a
        preconditioner replayed after convergence) and st is not written.
        local: a gs sub-plan to run instead of the rank-private segments
        (the fused CG update's >= 3-member segments, point_codes); w is then
        assembled only at those segments and the halo ids."""
        m = self.mesh
        L, s = lib(), stream_ptr()
        D = m.basis.diff  # host: passed by value to the kernel
        Bp = ptr(m.B) if self.lam1 != 0.0 else None
        g = self.gs
        multi = g.comm is not None and g.comm.size > 1

        def bk5(elems, base, reduce_count):
            nl = 0 if elems is None else int(elems.numel())
            check(L.nk_bk5(m.N, m.E, ptr(D), ptr(m.G), ptr(p), ptr(w), self.lam0, Bp, self.lam1,
                           self.ncomp, self.n, ptr(m.mask), ptr(elems), nl, ptr(st),
                           ptr(partials), base, reduce_count, s), "bk5")

        if not multi:
            nb = int(L.nk_bk5_blocks(m.N, m.E, self.ncomp))
            bk5(None, 0, nb if (st is not None and reduce) else 0)
            if self.ncomp == 1:
                _local(g, w, "+", 1, st=st)
            else:
                _local(g, w, "+", self.ncomp, st=st)
        else:
            import torch
            be, ie = g.boundary_elements, g.interior_elements
            nbb = int(L.nk_bk5_blocks(m.N, int(be.numel()), self.ncomp)) if be.numel() else 0
            nbi = int(L.nk_bk5_blocks(m.N, int(ie.numel()), self.ncomp)) if ie.numel() else 0
            if be.numel():
                bk5(be, 0, 0 if ie.numel() else (nbb if st is not None else 0))
            _halo_start(g, w, st=st)
            main = torch.cuda.current_stream()
            side = getattr(g, "_side", None)
            if side is None:
                side = g._side = torch.cuda.Stream(device=w.device)
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            with torch.cuda.stream(side):
                _halo_exchange(g)
                done = torch.cuda.Event()
                done.record(side)
            if ie.numel():
                bk5(ie, nbb, (nbb + nbi) if st is not None else 0)
            _local(g, w, "+", 1, st=st, part=g.seg_rest if local is None else local)
            main.wait_event(done)
            _halo_finish(g, w, "+", st=st)
        COUNTERS.add("stiffness", bk5_flops(m.N, m.E, self.ncomp), 7 * self.n * self.ncomp)
        return w

    def apply_pcg(self, p, w, x, r, invD, st, partials, hist, gs=True, local=None):
        """Fused BP5 operator step (nk_bk5_pcg): convergence test, deferred
        x += alpha p, Jacobi p = invD r + beta p, then w = A p with p^T A p
        into st->pAp -- followed by gs (and the halo on several ranks).
        gs=False (one rank) leaves w unassembled for nk_cg_update_gs; on
        several ranks `local` replaces the rank-private gs segments as in
        apply()."""
        m = self.mesh
        L, s = lib(), stream_ptr()
        D = m.basis.diff
        Bp = ptr(m.B) if self.lam1 != 0.0 else None
        g = self.gs
        multi = g.comm is not None and g.comm.size > 1

        def k1(elems, base, reduce_count):
            nl = 0 if elems is None else int(elems.numel())
            check(L.nk_bk5_pcg(m.N, m.E, ptr(D), ptr(m.G), ptr(p), ptr(w), self.lam0, Bp,
                               self.lam1, ptr(m.mask), ptr(elems), nl, ptr(x), ptr(r), ptr(invD),
                               ptr(st), ptr(partials), base, reduce_count, ptr(hist), s),
                  "bk5_pcg")

        if not multi:
            nb = int(L.nk_bk5_pcg_blocks(m.N, m.E))
            k1(None, 0, nb)
            if gs:
                _local(g, w, "+", 1, st=st)
        else:
            import torch
            be, ie = g.boundary_elements, g.interior_elements
            nbb = int(L.nk_bk5_pcg_blocks(m.N, int(be.numel()))) if be.numel() else 0
            nbi = int(L.nk_bk5_pcg_blocks(m.N, int(ie.numel()))) if ie.numel() else 0
            if be.numel():
                k1(be, 0, 0 if ie.numel() else nbb)
            _halo_start(g, w, st=st)
            main = torch.cuda.current_stream()
            side = getattr(g, "_side", None)
            if side is None:
                side = g._side = torch.cuda.Stream(device=w.device)
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            with torch.cuda.stream(side):
                _halo_exchange(g)
                done = torch.cuda.Event()
                done.record(side)
            if ie.numel():
                k1(ie, nbb, nbb + nbi)
            _local(g, w, "+", 1, st=st, part=g.seg_rest if local is None else local)
            main.wait_event(done)
            _halo_finish(g, w, "+", st=st)
        COUNTERS.add("stiffness", bk5_flops(m.N, m.E, 1), 7 * self.n)
        return w

    def partials_len(self):
        """Per-block partial slots for the fused p.Ap: one launch over all
        elements, or boundary + interior launches on several ranks (each can
        use a full persistent grid)."""
        m = self.mesh
        L = lib()
        g = self.gs
        sizes = [m.E]
        if g.comm is not None and g.comm.size > 1:
            sizes = [int(g.boundary_elements.numel()), int(g.interior_elements.numel())]
        tot_bk5 = sum(int(L.nk_bk5_blocks(m.N, n, self.ncomp)) for n in sizes if n)
        tot_pcg = sum(int(L.nk_bk5_pcg_blocks(m.N, n)) for n in sizes if n)
        return max(tot_bk5, tot_pcg, 1) + 2


class JacobiPreconditioner:
    """z = invD r with invD = mask / assembled diag(A)."""

    def __init__(self, op):
        self.op = op
        m = op.mesh
        d = extract_diagonal(m, spec=("helmholtz", op.lam0, op.lam1) if op.lam1 else "stiffness",
                             gs=op.gs)
        mask = m.mask.to(d.dtype)
        self.invD = (mask / d).reshape(-1).contiguous()

    def __call__(self, r, out=None):
        import torch
        if r.numel() != self.invD.numel():
            raise ContractError("contract error: field length mismatch")
        z = torch.empty_like(r) if out is None else out
        check(lib().nk_pointwise(r.numel(), ptr(self.invD), ptr(r), ptr(z), 1.0, None,
                                 stream_ptr()), "pointwise")
        return z


# orders whose fused BP5 step stays one kernel (N = 7: the TMA pipeline,
# 0.117 vs 0.138 ms split; N = 8, 9, 12: the stage kernel with the PCG head
# fused, 0.110 / 0.111 / 0.113 vs 0.118 / 0.118 / 0.120 ms split,
# profiles/r2zt_stage_pcg.jsonl); elsewhere FusedPCG splits it (split_step)
# once the rank's mesh is large enough that the 4th launch pays for itself:
# measured crossovers (scripts/split_crossover.py,
# profiles/r2zj_split_crossover*.jsonl, per-iteration time fused vs split):
# ~1-2M local points at N <= 5 (the split step is 10-30% SLOWER below),
# ~0.5-0.8M at N = 6..11, none at N >= 12.
SPLIT_STEP_OFF = (7, 8, 9, 12)


def split_min_points(N):
    """Local-point threshold of FusedPCG's automatic split_step rule."""
    if N >= 12:
        return 0
    return 2_000_000 if N <= 5 else 600_000


class FusedPCG:
    """Graph-captured Jacobi-PCG on a PoissonOperator (BP5).

    Buffers are allocated once; ``solve(b)`` runs init (2 launches + optional
    all-reduce), then replays a CUDA graph of ``chunk`` iterations until the
    device flag ``done`` is set.  Per iteration: nk_bk5_pcg (convergence
    test, deferred x update, Jacobi p update, BK5, p.Ap), gs, [halo],
    nk_cg_update (r, rr, rz, zAp).  On one rank the face pairs of the gs fold
    into the update (nk_cg_update_gs: a point of a 2-member segment adds its
    partner's w on the fly; the gs pass only covers edge / vertex segments)
    -- bit-identical; fuse_gs=False keeps the full gs pass.

    split_step (one rank, fused gs): run nk_bk5_pcg's vector head as its own
    coalesced pass (nk_cg_xpstep) followed by nk_bk5 with the fused p.Ap --
    4 kernels per iteration.  None = auto: on where it measured faster than
    the fused kernel -- every N not in SPLIT_STEP_OFF (7: the TMA pipeline;
    8, 9, 12: the stage kernel with the PCG head fused) once the mesh has
    split_min_points(N) local points
    (profiles/r2zj_split_crossover*.jsonl: 1.05-1.30x at the configs[1]
    sizes; below the crossover the fused step wins by up to 30%).

    gather_segments (one rank, fused gs; off by default): the update also
    folds the edge / vertex segments itself (nk_cg_update_gs_seg: every
    member of an M >= 3 segment gathers the segment in canonical order) --
    no gs pass, 2 kernels per iteration (3 split), bit-identical -- but
    measured SLOWER: 0.151 vs 0.115 ms per iteration at N = 7, E = 20^3
    (three dependent L2 round trips per warp trip for the ~16% edge /
    vertex points; profiles/r2j_bp5_knobs.jsonl)."""

    def __init__(self, op, prec, tol=1e-8, max_iter=1000, flexible=False, chunk=16,
                 use_graph=True, fuse_gs=True, split_step=None, gather_segments=False,
                 gs_tail=None):
        import torch
        self.op, self.prec = op, prec
        self.tol, self.max_iter, self.flexible = float(tol), int(max_iter), bool(flexible)
        self.chunk = max(1, int(chunk))
        comm = op.gs.comm
        board = False
        if comm is not None and comm.size > 1 and getattr(op.gs, "transport", "p2p") == "ipc":
            board = comm.enable_board(op.mesh.device)     # NCCL-free scalar all-reduce
        # graph capture needs every per-iteration exchange on the stream:
        # peer-memory halo + board, or NCCL (device staging)
        self.use_graph = use_graph and (comm is None or comm.size == 1 or board or
                                        comm.staging == "device")
        dev = op.mesh.device
        n = op.n * op.ncomp
        if op.ncomp != 1:
            raise ContractError("FusedPCG solves scalar fields; batch components with "
                                "one solver per component")
        self.n = n
        f = lambda: torch.zeros(n, dtype=torch.float64, device=dev)
        self.x, self.r, self.p, self.w = f(), f(), f(), f()
        self.st = _state_tensor(dev)
        self.part_bk5 = torch.zeros(op.partials_len(), dtype=torch.float64, device=dev)
        self.part_cg = torch.zeros(int(lib().nk_cg_partials_len(n)), dtype=torch.float64,
                                   device=dev)
        self.hist = torch.zeros(self.max_iter + 2, dtype=torch.float64, device=dev)
        # FP64 1/mult weights: measured slightly faster than the u8 multiplicity
        # option of nk_cg_update (latency- not byte-bound kernel)
        self.wt = op.weights
        self.mult = None
        self.invD = prec.invD
        self.comm = op.gs.comm if (op.gs.comm is not None and op.gs.comm.size > 1) else None
        self.s64 = self.st.view(torch.float64)   # rz pAp rz_new rr zap bb thresh2 alpha
        self.graph = None
        self.codes = None
        if fuse_gs:
            from .gather_scatter import point_codes
            self.codes = point_codes(op.gs)
        self.gcodes = None
        if fuse_gs and self.comm is None and gather_segments:
            from .gather_scatter import point_codes_gathered
            self.gcodes = point_codes_gathered(op.gs)
            if self.gcodes is not None and not _aligned16(self.r, self.w, self.invD):
                self.gcodes = None
        self.launches_per_iter = 3    # bk5_pcg, gs (all | non-pair segments), update
        if split_step is None:
            split_step = (op.mesh.N not in SPLIT_STEP_OFF and
                          op.mesh.n_local >= split_min_points(op.mesh.N))
        self.split = bool(split_step) and self.codes is not None
        if self.split:
            self.launches_per_iter = 4    # xpstep, bk5 (+p.Ap), gs non-pair, update
        if self.gcodes is not None:
            self.launches_per_iter -= 1   # no gs pass
        # the edge / vertex gs as the tail of the persistent step kernel
        # (nk_bk5_pcg_gs: one launch fewer, bit-identical; N = 7 TMA step,
        # NK_KNOB_GS_TAIL -- off by default: 5-7% slower per iteration in
        # graph replay, profiles/r2zzc_gs_tail_ab.jsonl)
        plan = self.codes[1] if self.codes is not None else None
        can_tail = (self.comm is None and not self.split and self.gcodes is None and
                    plan is not None and plan.rest is None and
                    bool(lib().nk_bk5_pcg_gs_fused(op.mesh.N)))
        self.gs_tail = can_tail if gs_tail is None else (bool(gs_tail) and can_tail)
        if self.gs_tail:
            self.launches_per_iter = 2    # bk5_pcg + gs tail, update
        elif (can_tail or (self.comm is None and self.gcodes is None and plan is not None and
                           plan.rest is None)) and lib().nk_cg_update_gs_cls_fused(n):
            self.launches_per_iter -= 1   # gs inside the update (NK_KNOB_GS_TAIL = 2)

    def _allreduce(self, a, b):
        if self.comm is not None:
            self.comm.allreduce_sum_(self.s64[a:b])

    def _iteration(self):
        """One PCG iteration = 3 kernels on one rank: nk_bk5_pcg (test,
        x/p updates, BK5, p.Ap), gs, nk_cg_update (r, rr, rz, zAp).  On
        several ranks the same with the boundary / interior BK5 split around
        the halo push, the combine, and the dot all-reduces."""
        L, s = lib(), stream_ptr()
        if self.codes is not None:
            if self.comm is not None:
                # private face pairs fold into the update; the >= 3-member
                # private segments run between the interior BK5 and the combine
                if self.split:
                    check(L.nk_cg_xpstep(self.n, ptr(self.x), ptr(self.r), ptr(self.p),
                                         ptr(self.invD), ptr(self.st), ptr(self.hist), s),
                          "cg_xpstep")
                    self.op.apply(self.p, self.w, self.st, self.part_bk5, local=self.codes[1])
                else:
                    self.op.apply_pcg(self.p, self.w, self.x, self.r, self.invD, self.st,
                                      self.part_bk5, self.hist, local=self.codes[1])
                self._allreduce(1, 2)                                    # pAp
                self._update_gs(L, s)
            elif self.gs_tail:
                self._step_gs_tail(L, s)
                self._update_gs(L, s)
            else:
                if self.split:
                    self._split_head(L, s)
                else:
                    self.op.apply_pcg(self.p, self.w, self.x, self.r, self.invD, self.st,
                                      self.part_bk5, self.hist, gs=False)
                self._gs_update(L, s)
            self._allreduce(2, 5)                                        # rz_new rr zap
            return
        self.op.apply_pcg(self.p, self.w, self.x, self.r, self.invD, self.st, self.part_bk5,
                          self.hist)
        self._allreduce(1, 2)                                            # pAp
        check(L.nk_cg_update(self.n, None, ptr(self.r), None, ptr(self.w), ptr(self.invD),
                             ptr(self.wt), ptr(self.mult), ptr(self.st), ptr(self.part_cg), s),
              "cg_update")
        self._allreduce(2, 5)                                            # rz_new rr zap

    def _step_gs_tail(self, L, s):
        """nk_bk5_pcg_gs: the fused step with the >= 3-member gs folded into
        its tail after a grid barrier (same bits as nk_bk5_pcg + the gs pass)."""
        op, m, pl = self.op, self.op.mesh, self.codes[1]
        nb = int(L.nk_bk5_pcg_blocks(m.N, m.E))
        check(L.nk_bk5_pcg_gs(m.N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(self.p), ptr(self.w),
                              op.lam0, ptr(m.B) if op.lam1 != 0.0 else None, op.lam1,
                              ptr(m.mask), ptr(self.x), ptr(self.r), ptr(self.invD),
                              ptr(self.st), ptr(self.part_bk5), nb, ptr(self.hist),
                              pl.nclass, ptr(pl.sizes), ptr(pl.nsegs), ptr(pl.ptrs), s),
              "bk5_pcg_gs")

    def _edge_vertex_gs(self):
        """The gs pass over the >= 3-member segments, unless the update
        gathers them itself."""
        if self.gcodes is None:
            self.codes[1].run(self.w, "+", 1, self.n, self.st)

    def _gs_update(self, L, s):
        """The edge / vertex gs pass + the update: nk_cg_update_gs_cls (one
        launch under NK_KNOB_GS_TAIL = 2, else the same two launches)."""
        pl = self.codes[1]
        if self.gcodes is not None or pl.rest is not None:
            self._edge_vertex_gs()
            self._update_gs(L, s)
            return
        check(L.nk_cg_update_gs_cls(self.n, ptr(self.r), ptr(self.w), ptr(self.invD),
                                    ptr(self.codes[0]), pl.nclass, ptr(pl.sizes), ptr(pl.nsegs),
                                    ptr(pl.ptrs), ptr(self.st), ptr(self.part_cg), s),
              "cg_update_gs_cls")

    def _update_gs(self, L, s):
        """nk_cg_update_gs (face pairs folded in) or, with gathered segments,
        nk_cg_update_gs_seg (every shared point assembled in the update)."""
        if self.gcodes is not None:
            check(L.nk_cg_update_gs_seg(self.n, 1, 0, ptr(self.r), ptr(self.w), ptr(self.invD),
                                        ptr(self.gcodes[0]), ptr(self.gcodes[1]), ptr(self.st),
                                        ptr(self.part_cg), s), "cg_update_gs_seg")
        else:
            check(L.nk_cg_update_gs(self.n, ptr(self.r), ptr(self.w), ptr(self.invD),
                                    ptr(self.codes[0]), ptr(self.st), ptr(self.part_cg), s),
                  "cg_update_gs")

    def _split_head(self, L, s, mid_event=None):
        """nk_cg_xpstep (test, x and p updates) + nk_bk5 with the fused p.Ap:
        the same iterates as nk_bk5_pcg up to the rounding of the BK5
        variant the order's table picks.  mid_event (profiling) is recorded
        between the two launches."""
        op, m = self.op, self.op.mesh
        check(L.nk_cg_xpstep(self.n, ptr(self.x), ptr(self.r), ptr(self.p), ptr(self.invD),
                             ptr(self.st), ptr(self.hist), s), "cg_xpstep")
        if mid_event is not None:
            mid_event.record()
        nb = int(L.nk_bk5_blocks(m.N, m.E, 1))
        check(L.nk_bk5(m.N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(self.p), ptr(self.w),
                       op.lam0, ptr(m.B) if op.lam1 else None, op.lam1, 1, self.n, ptr(m.mask),
                       None, 0, ptr(self.st), ptr(self.part_bk5), 0, nb, s), "bk5")
        COUNTERS.add("stiffness", bk5_flops(m.N, m.E, 1), 7 * self.n)

    def _capture(self):
        import torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(self.chunk):
                self._iteration()
        self.graph = g

    def profile_iteration(self, reps=20):
        """In-situ device time (ms) of each kernel group of one iteration,
        CUDA events between launches on the current stream (eager, no graph;
        L2 state as in a real solve).  Returns {name: ms}.  Not counted in
        KernelCounters (measurement replays)."""
        with COUNTERS.recording():
            return self._profile_iteration(reps)

    def _profile_iteration(self, reps):
        import torch
        L, s = lib(), stream_ptr()
        op, g = self.op, self.op.gs
        fused = self.codes is not None
        split = fused and self.split
        names = ("bk5_pcg", "gs_nonpair", "cg_update_gs") if fused else ("bk5_pcg", "gs", "cg_update")
        if split:
            names = ("cg_xpstep", "bk5") + names[1:]
        acc = dict.fromkeys(names, 0.0)
        st_save = self.st.clone()
        m = op.mesh
        for _ in range(reps):
            self.st.copy_(st_save)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
            ev0 = ev[0]
            ev[0].record()
            if split:
                self._split_head(L, s, mid_event=ev[1])
                ev = ev[1:]   # the remaining indices line up with the 3-kernel form
            elif self.gs_tail:
                self._step_gs_tail(L, s)
            else:
                nb = int(L.nk_bk5_pcg_blocks(m.N, m.E))
                check(L.nk_bk5_pcg(m.N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(self.p),
                                   ptr(self.w), op.lam0, ptr(m.B) if op.lam1 else None, op.lam1,
                                   ptr(m.mask), None, 0, ptr(self.x), ptr(self.r),
                                   ptr(self.invD), ptr(self.st), ptr(self.part_bk5), 0, nb,
                                   ptr(self.hist), s), "bk5_pcg")
            ev[1].record()
            if fused:
                if not self.gs_tail:
                    self._edge_vertex_gs()
                ev[2].record()
                self._update_gs(L, s)
                ev[3].record()
            else:
                _local(g, self.w, "+", 1, st=self.st)
                ev[2].record()
                check(L.nk_cg_update(self.n, None, ptr(self.r), None, ptr(self.w),
                                     ptr(self.invD), ptr(self.wt), ptr(self.mult), ptr(self.st),
                                     ptr(self.part_cg), s), "cg_update")
                ev[3].record()
            torch.cuda.synchronize()
            if split:
                ev = [ev0] + ev
            for q, nm in enumerate(names):
                acc[nm] += ev[q].elapsed_time(ev[q + 1])
        self.st.copy_(st_save)
        if self.gcodes is not None or self.gs_tail:
            acc.pop("gs_nonpair")    # folded into the update / the step's tail
        return {k: v / reps for k, v in acc.items()}

    def init(self, b):
        L, s = lib(), stream_ptr()
        # init always uses the FP64 weights (exactly 1/mult, equal to the u8 path)
        check(L.nk_cg_init(self.n, ptr(b), ptr(self.x), ptr(self.r), ptr(self.p),
                           ptr(self.invD), ptr(self.op.weights), ptr(self.st), ptr(self.part_cg),
                           self.tol, self.max_iter, int(self.flexible), s), "cg_init")
        self._allreduce(0, 1)   # rz
        self._allreduce(3, 4)   # rr
        self._allreduce(5, 6)   # bb
        check(L.nk_cg_init_finalize(ptr(self.st), ptr(self.hist), s), "cg_init_finalize")

    def run(self, sync_every=None):
        """Iterate until done; returns the host copy of the state."""
        import torch
        if self.use_graph and self.graph is None:
            # capture while done == 1 would still record the kernels; capture
            # is independent of the state values.  The counters of one
            # captured chunk are kept and added per executed iteration.
            with COUNTERS.recording() as rec:
                self._capture()
            self._iter_counts = (rec, self.chunk)
        done_h = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        off = CGState.done.offset
        done_dev = self.st[off:off + 4].view(torch.int32)
        while True:
            if self.use_graph:
                self.graph.replay()
            else:
                with COUNTERS.recording() as rec:
                    for _ in range(self.chunk):
                        self._iteration()
                self._iter_counts = (rec, self.chunk)
            done_h.copy_(done_dev, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            if int(done_h[0]):
                break
        return read_state(self.st)

    def solve(self, b):
        import torch
        if not isinstance(b, torch.Tensor):
            raise ContractError("b must be a CUDA tensor")
        bb = b.reshape(-1)
        if bb.numel() != self.n or bb.dtype != torch.float64 or not bb.is_cuda:
            raise ContractError("contract error: rhs length/dtype mismatch")
        self.init(bb.contiguous())
        stt = self.run()
        if stt.breakdown:
            raise BreakdownError(f"p^T A p <= 0 at iteration {stt.iter}")
        it = int(stt.iter)
        _count_iterations(self, it)
        hist = self.hist[:it + 1].cpu().numpy().tolist()
        return PCGResult(self.x.view_as(b), it, hist, bool(stt.converged))


def _count_iterations(solver, it):
    """KernelCounters for a graph-captured / chunked solve: the counts of one
    recorded chunk, scaled to the iterations that ran (exact: every
    iteration issues the same launches)."""
    ic = getattr(solver, "_iter_counts", None)
    if ic is not None:
        COUNTERS.add_scaled(ic[0], it, ic[1])


def pcg(apply_A, apply_M, b, tol=1e-8, max_iter=1000, flexible=False, weights=None, x0=None,
        chunk=16):
    """PCG.  Returns PCGResult(x, iterations,
    residual_history, converged).  b: CUDA float64 tensor (or numpy ->
    numpy x).  weights: per-entry dot weights (default: the operator's
    1/multiplicity for a PoissonOperator, else ones)."""
    import torch
    host = isinstance(b, np.ndarray)
    if isinstance(apply_A, PoissonOperator):
        dev = apply_A.mesh.device
    else:
        dev = b.device if isinstance(b, torch.Tensor) else "cuda"
    bt = torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64), device=dev) if host else b
    if (isinstance(apply_A, PoissonOperator) and isinstance(apply_M, JacobiPreconditioner)
            and apply_M.op is apply_A and x0 is None and weights is None and apply_A.ncomp == 1):
        res = FusedPCG(apply_A, apply_M, tol, max_iter, flexible, chunk=chunk).solve(bt)
        if host:
            res = res._replace(x=res.x.cpu().numpy().reshape(np.shape(b)))
        return res
    from .multigrid import MultigridHierarchy, MultigridPCG
    if (isinstance(apply_A, PoissonOperator) and isinstance(apply_M, MultigridHierarchy)
            and apply_M.levels[0].op is apply_A and x0 is None and weights is None):
        res = MultigridPCG(apply_A, apply_M, tol, max_iter, flexible).solve(bt)
        if host:
            res = res._replace(x=res.x.cpu().numpy().reshape(np.shape(b)))
        return res
    return _pcg_generic(apply_A, apply_M, bt, tol, max_iter, flexible, weights, x0, host,
                        np.shape(b))


def _pcg_generic(apply_A, apply_M, b, tol, max_iter, flexible, weights, x0, host, shape):
    import torch
    L = lib()
    dev = b.device
    n = b.numel()
    flat = lambda t: t.reshape(-1)
    if weights is None and isinstance(apply_A, PoissonOperator):
        weights = apply_A.weights
    wt = None if weights is None else flat(torch.as_tensor(weights, dtype=torch.float64,
                                                           device=dev)).contiguous()
    st = _state_tensor(dev)
    s64 = st.view(torch.float64)
    part = torch.zeros(int(L.nk_cg_partials_len(n)), dtype=torch.float64, device=dev)
    hist = torch.zeros(max_iter + 2, dtype=torch.float64, device=dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    r = torch.zeros_like(x)
    p = torch.zeros_like(x)
    s = stream_ptr()
    bf = flat(b).contiguous()
    if x0 is not None:
        x0t = flat(torch.as_tensor(np.asarray(x0) if not isinstance(x0, torch.Tensor) else x0,
                                   dtype=torch.float64, device=dev)).contiguous()
        rhs = (bf - flat(apply_A(x0t.view_as(b)))).contiguous()
    else:
        x0t, rhs = None, bf
    # init with invD = NULL: p = r, then replace p by M r and recompute rz
    check(L.nk_cg_init(n, ptr(rhs), ptr(x), ptr(r), ptr(p), None, ptr(wt), ptr(st), ptr(part),
                       tol, max_iter, int(flexible), s), "cg_init")
    # the stopping test is relative to ||b||, not to the initial residual
    check(L.nk_wdot(n, ptr(bf), ptr(bf), ptr(wt), ptr(s64[5:6]), ptr(part), s), "wdot")
    z = flat(apply_M(r.view_as(b))).contiguous()
    p.copy_(z)
    check(L.nk_wdot(n, ptr(r), ptr(z), ptr(wt), ptr(s64[0:1]), ptr(part), s), "wdot")
    check(L.nk_cg_init_finalize(ptr(st), ptr(hist), s), "cg_init_finalize")
    stt = read_state(st)
    Ap = torch.zeros_like(x)
    while not stt.done:
        Ap = flat(apply_A(p.view_as(b))).contiguous()
        check(L.nk_wdot(n, ptr(p), ptr(Ap), ptr(wt), ptr(s64[1:2]), ptr(part), s), "wdot")
        check(L.nk_cg_update(n, ptr(x), ptr(r), ptr(p), ptr(Ap), None, ptr(wt), None, ptr(st),
                             ptr(part), s), "cg_update")
        z = flat(apply_M(r.view_as(b))).contiguous()
        check(L.nk_wdot(n, ptr(r), ptr(z), ptr(wt), ptr(s64[2:3]), ptr(part), s), "wdot")
        if flexible:
            check(L.nk_wdot(n, ptr(z), ptr(Ap), ptr(wt), ptr(s64[4:5]), ptr(part), s), "wdot")
        check(L.nk_cg_pupdate(n, ptr(r), ptr(p), None, ptr(z), ptr(st), ptr(hist), s),
              "cg_pupdate")
        stt = read_state(st)
    if stt.breakdown:
        raise BreakdownError(f"p^T A p <= 0 at iteration {stt.iter}")
    if x0t is not None:
        x += x0t
    it = int(stt.iter)
    xo = x.view_as(b)
    res = PCGResult(xo.cpu().numpy().reshape(shape) if host else xo, it,
                    hist[:it + 1].cpu().numpy().tolist(), bool(stt.converged))
    return res


class FusedPCG3:
    """Lockstep batched Jacobi-PCG for three right-hand sides of ONE operator
    (the vector Helmholtz solve, configs[4]; "geometric
    factors ... reused across each velocity component").

    Three independent CG states advance together, one launch per stage for
    all three components (4 kernels per iteration for three solves):
      nk_cg_xpstep_batch   per-component stop test, deferred x update,
                           Jacobi p update (gridDim.y = component);
      nk_bk5_batch         w_c = mask A p_c with p_c . A p_c per component --
                           the seq3 kernel reads G from HBM ONCE for the
                           three components (orders where the measured table
                           picks it; three scalar launches elsewhere);
      gs sub-plan          edge / vertex segments, ncomp = 3;
      nk_cg_update_gs_batch  face pairs folded in, r_c, rr_c, rz_c, zAp_c.
    Each component keeps its own scalars, iteration count, residual history
    and convergence; a converged component's launches are no-ops (its BK5
    part is skipped inside the kernel).  The iterates of component c are
    those of a scalar FusedPCG solve of b_c up to the BK5 kernel's rounding
    (same algorithm, same reductions).  One rank (several ranks: solve the
    components one by one with FusedPCG)."""

    NC = 3

    def __init__(self, op, prec, tol=1e-6, max_iter=1000, flexible=False, chunk=16,
                 use_graph=True, gather_segments=False):
        import torch
        from .gather_scatter import point_codes, point_codes_gathered
        if op.gs.comm is not None and op.gs.comm.size > 1:
            raise ContractError("FusedPCG3 runs on one rank")
        if op.ncomp != 1:
            raise ContractError("FusedPCG3 takes the scalar operator (one per component)")
        self.op, self.prec = op, prec
        self.tol, self.max_iter, self.flexible = float(tol), int(max_iter), bool(flexible)
        self.chunk = max(1, int(chunk))
        self.use_graph = bool(use_graph)
        m = op.mesh
        dev = m.device
        n = self.n = op.n
        L = lib()
        f = lambda: torch.zeros(self.NC * n, dtype=torch.float64, device=dev)
        self.x, self.r, self.p, self.w = f(), f(), f(), f()
        self.st = torch.zeros(self.NC * CG_STATE_BYTES, dtype=torch.uint8, device=dev)
        self.pstride = int(L.nk_bk5_batch_blocks(m.N, m.E)) + 2
        self.part_bk5 = torch.zeros(self.NC * self.pstride, dtype=torch.float64, device=dev)
        self.cg_plen = int(L.nk_cg_partials_len(n))
        self.part_cg = torch.zeros(self.NC * self.cg_plen, dtype=torch.float64, device=dev)
        self.hstride = self.max_iter + 2
        self.hist = torch.zeros(self.NC * self.hstride, dtype=torch.float64, device=dev)
        self.invD = prec.invD
        self.codes = point_codes(op.gs)
        if self.codes is None:
            raise ContractError("FusedPCG3 needs n < 2^31 local points")
        # gathered segments: the update folds edges / vertices itself (no gs pass)
        self.gcodes = point_codes_gathered(op.gs) if gather_segments else None
        self.graph = None
        self.variant = int(L.nk_bk5_batch_variant(m.N))
        self.launches_per_iter = (4 if self.variant == 6 else 6) - (self.gcodes is not None)

    def _update(self, L, s):
        n = self.n
        if self.gcodes is not None:
            check(L.nk_cg_update_gs_seg(n, self.NC, n, ptr(self.r), ptr(self.w), ptr(self.invD),
                                        ptr(self.gcodes[0]), ptr(self.gcodes[1]), ptr(self.st),
                                        ptr(self.part_cg), s), "cg_update_gs_seg")
            return
        self.codes[1].run(self.w, "+", self.NC, n)                     # edges, vertices
        check(L.nk_cg_update_gs_batch(n, self.NC, n, ptr(self.r), ptr(self.w), ptr(self.invD),
                                      ptr(self.codes[0]), ptr(self.st), ptr(self.part_cg), s),
              "cg_update_gs_batch")

    def _sti(self, c):
        return self.st.data_ptr() + c * CG_STATE_BYTES

    def _iteration(self):
        L, s = lib(), stream_ptr()
        op, m = self.op, self.op.mesh
        n = self.n
        check(L.nk_cg_xpstep_batch(n, self.NC, n, ptr(self.x), ptr(self.r), ptr(self.p),
                                   ptr(self.invD), ptr(self.st), ptr(self.hist), self.hstride, s),
              "cg_xpstep_batch")
        nb = self.pstride - 2
        check(L.nk_bk5_batch(m.N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(self.p), ptr(self.w),
                             op.lam0, ptr(m.B) if op.lam1 else None, op.lam1, self.NC, n,
                             ptr(m.mask), None, 0, ptr(self.st), ptr(self.part_bk5), self.pstride,
                             0, nb, s), "bk5_batch")
        COUNTERS.add("stiffness", bk5_flops(m.N, m.E, self.NC), 7 * n * self.NC)
        self._update(L, s)

    def profile_iteration(self, b3, reps=10):
        """In-situ device time (ms) of each stage of one batched iteration
        (CUDA events between launches, eager; state restored between reps):
        {'xpstep', 'bk5', 'gs_nonpair', 'update_gs'}."""
        import torch
        L, s = lib(), stream_ptr()
        op, m = self.op, self.op.mesh
        n = self.n
        names = ("xpstep", "bk5", "gs_nonpair", "update_gs")
        acc = dict.fromkeys(names, 0.0)
        with COUNTERS.recording():
            self.init(b3.reshape(-1).contiguous())
            for _ in range(2):
                self._iteration()
            save = [t.clone() for t in (self.st, self.x, self.r, self.p)]
            for _ in range(reps):
                for t, v in zip((self.st, self.x, self.r, self.p), save):
                    t.copy_(v)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                ev[0].record()
                check(L.nk_cg_xpstep_batch(n, self.NC, n, ptr(self.x), ptr(self.r), ptr(self.p),
                                           ptr(self.invD), ptr(self.st), ptr(self.hist),
                                           self.hstride, s), "xpstep")
                ev[1].record()
                check(L.nk_bk5_batch(m.N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(self.p),
                                     ptr(self.w), op.lam0, ptr(m.B) if op.lam1 else None,
                                     op.lam1, self.NC, n, ptr(m.mask), None, 0, ptr(self.st),
                                     ptr(self.part_bk5), self.pstride, 0, self.pstride - 2, s),
                      "bk5_batch")
                ev[2].record()
                if self.gcodes is None:
                    self.codes[1].run(self.w, "+", self.NC, n)
                ev[3].record()
                if self.gcodes is not None:
                    self._update(L, s)
                else:
                    check(L.nk_cg_update_gs_batch(n, self.NC, n, ptr(self.r), ptr(self.w),
                                                  ptr(self.invD), ptr(self.codes[0]),
                                                  ptr(self.st), ptr(self.part_cg), s), "update")
                ev[4].record()
                torch.cuda.synchronize()
                for q, nm in enumerate(names):
                    acc[nm] += ev[q].elapsed_time(ev[q + 1])
        return {k: v / reps for k, v in acc.items()}

    def init(self, b3):
        L, s = lib(), stream_ptr()
        n = self.n
        wt = self.op.weights
        for c in range(self.NC):
            o = c * n
            check(L.nk_cg_init(n, ptr(b3[o:o + n]), ptr(self.x[o:o + n]), ptr(self.r[o:o + n]),
                               ptr(self.p[o:o + n]), ptr(self.invD), ptr(wt), self._sti(c),
                               ptr(self.part_cg), self.tol, self.max_iter, int(self.flexible), s),
                  "cg_init")
            check(L.nk_cg_init_finalize(self._sti(c), ptr(self.hist[c * self.hstride:]), s),
                  "cg_init_finalize")

    def _done(self):
        import torch
        off = CGState.done.offset
        v = self.st.view(self.NC, CG_STATE_BYTES)[:, off:off + 4].contiguous()
        return bool(torch.all(v.view(torch.int32) != 0))

    def run(self):
        import torch
        if self.use_graph and self.graph is None:
            with COUNTERS.recording() as rec:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(self.chunk):
                        self._iteration()
                self.graph = g
            self._per_iter = (rec, self.chunk)
        while not self._done():
            if self.use_graph:
                self.graph.replay()
            else:
                with COUNTERS.recording() as rec:
                    for _ in range(self.chunk):
                        self._iteration()
                self._per_iter = (rec, self.chunk)
        raw = self.st.cpu().numpy().tobytes()
        return [CGState.from_buffer_copy(raw[c * CG_STATE_BYTES:(c + 1) * CG_STATE_BYTES])
                for c in range(self.NC)]

    def solve(self, b3):
        """b3: 3 component-major CUDA float64 fields (assembled, masked), any
        shape with 3 * n entries.  Returns (x3 view shaped like b3, [PCGResult
        per component]); x3 is the solver's buffer (overwritten next solve)."""
        import torch
        if not isinstance(b3, torch.Tensor) or not b3.is_cuda or b3.dtype != torch.float64 \
                or b3.numel() != self.NC * self.n:
            raise ContractError("contract error: rhs must be 3 x n CUDA float64")
        self.init(b3.reshape(-1).contiguous())
        sts = self.run()
        results = []
        x3 = self.x.view_as(b3)
        for c, stt in enumerate(sts):
            if stt.breakdown:
                raise BreakdownError(f"component {c}: p^T A p <= 0 at iteration {stt.iter}")
            it = int(stt.iter)
            hist = self.hist[c * self.hstride:c * self.hstride + it + 1].cpu().numpy().tolist()
            results.append(PCGResult(x3[c], it, hist, bool(stt.converged)))
        # counters: one stiffness application per component iteration
        rec, chunk = self._per_iter
        per_comp = {k: v // (chunk * self.NC) for k, v in rec.flops.items()}
        refs = {k: v // (chunk * self.NC) for k, v in rec.memory_refs.items()}
        tot = sum(r.iterations for r in results)
        for k in per_comp:
            COUNTERS.add(k, per_comp[k] * tot, refs[k] * tot)
        return x3, results


# orders where the lockstep 3-component PCG beats three scalar solves
BATCHED_HELM3_ORDERS = (10, 11, 12, 13)


class HelmholtzVectorSolver:
    """Viscous substep solve:
    per-component Jacobi-PCG on H = lam0 A + lam1 B, e.g. lam0 = 1/Re,
    lam1 = beta0/dt, for a 3-component (component-major) velocity field.
    One operator, one Jacobi diagonal and one set of fused-PCG buffers are
    shared by the components; each component is an independent FusedPCG
    solve (its own scalars, convergence and iteration count).
    ``apply(u3)`` is the batched operator (G read once for all components)."""

    def __init__(self, mesh, lam0, lam1, gs=None, comm=None, tol=1e-6, max_iter=1000,
                 chunk=16, batched=None):
        self.op = PoissonOperator(mesh, gs=gs, lam0=lam0, lam1=lam1, comm=comm)
        self.jac = JacobiPreconditioner(self.op)
        self.tol, self.max_iter, self.chunk = tol, max_iter, chunk
        multi = self.op.gs.comm is not None and self.op.gs.comm.size > 1
        # batched (FusedPCG3, lockstep, G once per iteration for the three
        # components): one rank, at the orders where it measured faster than
        # three scalar FusedPCG solves -- the scalar step carries the round-2
        # kernels (TMA step at N = 7, stage step with the fused PCG head,
        # pipelined gs update), which outweigh reading G three times except
        # at N = 10..13 (profiles/r2zz_helm3_batched_vs_seq.jsonl: e.g.
        # configs[4], N = 9: 233 vs 249 ms; N = 12: 73 vs 70 ms); several
        # ranks solve the components in turn
        self.batched = ((not multi and mesh.N in BATCHED_HELM3_ORDERS) if batched is None
                        else bool(batched))
        self._solver = None
        self.mesh = mesh

    @property
    def solver(self):
        if self._solver is None:
            cls = FusedPCG3 if self.batched else FusedPCG
            self._solver = cls(self.op, self.jac, tol=self.tol, max_iter=self.max_iter,
                               chunk=self.chunk)
        return self._solver

    def apply(self, u3, out=None):
        """w_c = mask * QQ^T (lam0 A_L + lam1 B) u_c for c = 0, 1, 2."""
        import torch
        from .gather_scatter import _local
        from .kernels import _as_device, _bk5
        m = self.mesh
        t, host = _as_device(u3, m, 3)
        # the Dirichlet mask is fused into the BK5 epilogue: it is continuous
        # (equal on every copy of an id), so mask QQ^T w = QQ^T (mask w)
        w = _bk5(t, m, self.op.lam0, self.op.lam1, 3, out=out, mask=True)
        g = self.op.gs
        if g.comm is not None and g.comm.size > 1:
            for c in range(3):
                gs_op(g, w.view(3, -1)[c])
        else:
            _local(g, w, "+", 3)
        return w.cpu().numpy().reshape(np.shape(u3)) if host else w

    def solve(self, b3):
        """b3: (3, E, nq, nq, nq) CUDA float64 (assembled, masked).  Returns
        (x3, [PCGResult per component])."""
        import torch
        x3 = torch.empty_like(b3)
        if self.batched:
            xs, results = self.solver.solve(b3)
            x3.copy_(xs)
            return x3, [r._replace(x=x3[c]) for c, r in enumerate(results)]
        results = []
        for c in range(3):
            r = self.solver.solve(b3[c].contiguous())
            x3[c].copy_(r.x)
            results.append(r._replace(x=x3[c]))
        return x3, results
