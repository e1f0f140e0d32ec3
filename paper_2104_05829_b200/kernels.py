"""Element-local operators -- the drop-in for the hot-path part of
``nekmini.kernels``.

apply_stiffness_local is the BK5 kernel (nk_bk5, csrc/bk5_*.cu); the
Helmholtz form lam0*A + lam1*B and the
3-component batch (G read once for u, v, w) use the same launch.
"""

from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np

from ._lib import ContractError, check, lib, ptr, stream_ptr

__all__ = ["apply_stiffness_local", "apply_helmholtz_local", "apply_mass", "inner_product",
           "extract_diagonal", "KernelCounters", "COUNTERS", "bk5_bytes", "bk5_flops",
           "select_kernel_variant", "reset_kernel_variant", "variant_report", "BK5_VARIANTS"]


@dataclass
class KernelCounters:
    """Formula-based counters: semantic, not
    hardware.  flops/memory_refs per kernel class."""
    flops: dict = field(default_factory=dict)
    memory_refs: dict = field(default_factory=dict)

    def add(self, name, flops, refs):
        self.flops[name] = self.flops.get(name, 0) + int(flops)
        self.memory_refs[name] = self.memory_refs.get(name, 0) + int(refs)

    def reset(self):
        self.flops.clear()
        self.memory_refs.clear()

    @contextmanager
    def recording(self):
        """Divert adds into a fresh KernelCounters (yielded) for the duration:
        graph-captured solvers record one captured iteration's counts here and
        add them once per iteration actually executed (add_scaled), so the
        totals count device work, not captures or no-op replays."""
        saved = (self.flops, self.memory_refs)
        rec = KernelCounters()
        self.flops, self.memory_refs = rec.flops, rec.memory_refs
        try:
            yield rec
        finally:
            self.flops, self.memory_refs = saved

    def add_scaled(self, other, num, den=1):
        """self += other * num / den (exact integer arithmetic)."""
        for k, v in other.flops.items():
            self.flops[k] = self.flops.get(k, 0) + v * int(num) // int(den)
        for k, v in other.memory_refs.items():
            self.memory_refs[k] = self.memory_refs.get(k, 0) + v * int(num) // int(den)


COUNTERS = KernelCounters()


def bk5_flops(N, E, ncomp=1):
    """12(N+1)^4 + 15(N+1)^3 flops per element."""
    nq = N + 1
    return ncomp * E * (12 * nq ** 4 + 15 * nq ** 3)


def bk5_bytes(N, E, ncomp=1, mass=False, mask=False):
    """Algorithmic HBM bytes of one BK5 launch: u + w per component, six G
    factors once, plus B (8) and mask (1) when used."""
    pts = E * (N + 1) ** 3
    return pts * (16 * ncomp + 48 + (8 if mass else 0) + (1 if mask else 0))


def _as_device(u, mesh, ncomp):
    import torch
    if isinstance(u, np.ndarray):
        return torch.as_tensor(np.ascontiguousarray(u, dtype=np.float64),
                               device=mesh.device), True
    if not isinstance(u, torch.Tensor) or not u.is_cuda or u.dtype != torch.float64:
        raise ContractError("field must be a CUDA float64 tensor or a numpy array")
    return u.contiguous(), False


def _bk5(u, mesh, lam0, lam1, ncomp, out=None, elements=None, mask=False, st=None,
         partials=None, part_base=0, reduce_count=0):
    import torch
    nloc = mesh.n_local
    if u.numel() != nloc * ncomp:
        raise ContractError(f"contract error: field length {u.numel()} != {nloc * ncomp}")
    w = torch.empty_like(u) if out is None else out
    if elements is not None and elements.numel() == 0:
        return w            # empty subset (its data pointer is NULL = "all" in the ABI)
    D = mesh.basis.diff  # host array: baked into the launch parameters
    nl = 0 if elements is None else int(elements.numel())
    check(lib().nk_bk5(mesh.N, mesh.E, ptr(D), ptr(mesh.G), ptr(u), ptr(w), float(lam0),
                       ptr(mesh.B) if lam1 != 0.0 else None, float(lam1), ncomp, nloc,
                       ptr(mesh.mask) if mask else None, ptr(elements), nl, ptr(st),
                       ptr(partials), part_base, reduce_count, stream_ptr()), "bk5")
    E = mesh.E if elements is None else nl
    COUNTERS.add("stiffness", bk5_flops(mesh.N, E, ncomp), 7 * E * mesh.nq ** 3 * ncomp)
    return w


def _is_host(u):
    import torch
    return isinstance(u, np.ndarray) or (isinstance(u, torch.Tensor) and not u.is_cuda)


class _HostStream:
    """Chunked host<->device pipeline for fields that live in host memory:
    chunk c's H2D (copy-in stream), BK5 (compute stream) and D2H (copy-out
    stream) overlap with neighbouring chunks, so the apply runs at the PCIe
    rate of max(H2D, D2H) instead of H2D + kernel + D2H.  Staging buffers are
    pinned and device buffers are reused across calls (per mesh).

    Measured alternatives (scripts/e2e_chunks.py, E = 8000, N = 7): the BK5
    reading u / writing w directly in pinned host memory (zero-copy) costs
    0.93 ms with the k-slab kernel (coalesced 128-B PCIe transactions) and
    2.5 ms with the pencil kernels (16-B pieces); copy-engine H2D + k-slab
    writing w straight to host is 0.85-0.88 ms on a warm L2 but 0.99 ms under
    bench.py's cold-L2 protocol, vs 0.90 ms for this pipeline (floor: 0.66-0.74
    ms for concurrent H2D + D2H copies of the same bytes).

    direct (round 2, orders in DIRECT_ORDERS, pinned buffers): copy-engine H2D
    per chunk, and the stage kernel (bk5_stage.cuh) writes each chunk's w
    straight into the pinned host buffer with its cp.async.bulk stores -- whole
    4-KB element images over PCIe, no D2H copies and no copy-out tail:
    0.855 ms with 8 chunks vs 0.902 ms for the copy pipeline at N = 7 under
    bench.py's cold-L2 protocol (scripts/e2e_ab.py, profiles/r2zl_e2e_ab.json),
    bit-identical."""

    DIRECT_ORDERS = (7,)
    # direct mode as ONE chunk-gated stage kernel (nk_bk5_set_gate) instead of
    # one kernel per chunk: correct, measured slower (0.883 vs 0.860 ms at 8
    # chunks, worse with more chunks: every chunk boundary stalls each
    # persistent CTA on the arrival frontier; profiles/r2zw_e2e_stream.json)
    STREAM = False

    def __init__(self, mesh, nchunks):
        import torch
        self.mesh, self.nchunks = mesh, nchunks
        self.direct = mesh.N in self.DIRECT_ORDERS
        n = mesh.n_local
        self.ud = torch.empty(n, dtype=torch.float64, device=mesh.device)
        self.wd = torch.empty(n, dtype=torch.float64, device=mesh.device)
        self.s_in, self.s_cmp, self.s_out = (torch.cuda.Stream(device=mesh.device) for _ in range(3))
        self.graphs = {}
        # stream mode: the device gate the kernel polls (element count of the
        # H2D chunks landed so far)
        self.gate = torch.zeros(1, dtype=torch.int64, device=mesh.device)

    def run(self, uh, wh, use_graph=True):
        """uh, wh: contiguous float64 host tensors.  Pinned buffers: the whole
        chunk pipeline is captured once per (uh, wh) pair as a CUDA graph
        (fork to three streams, memcpy + BK5 nodes, join) and replayed, so
        the chunk count costs no host time."""
        import torch
        if use_graph and uh.is_pinned() and wh.is_pinned():
            key = (uh.data_ptr(), wh.data_ptr(), uh.numel())
            g = self.graphs.get(key)
            if g is None:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._issue(uh, wh)
                self.graphs[key] = g
            g.replay()
            COUNTERS.add("stiffness", bk5_flops(self.mesh.N, self.mesh.E), 7 * self.mesh.n_local)
            return wh
        self._issue(uh, wh)
        COUNTERS.add("stiffness", bk5_flops(self.mesh.N, self.mesh.E), 7 * self.mesh.n_local)
        return wh

    def _bounds(self, E):
        """Tapered chunks: small first and last chunks keep the exposed
        head H2D and tail D2H short; large middle chunks amortise per-copy
        costs.  nchunks = 4 -> sizes proportional to 1, 3, 3, 1 (etc.)."""
        k = self.nchunks
        if k <= 2:
            w = np.ones(k)
        else:
            w = np.minimum(np.arange(1, k + 1), np.arange(k, 0, -1)).astype(float)
            w = np.minimum(w * 2 - 1, 4.0)
        c = np.concatenate([[0.0], np.cumsum(w) / w.sum()])
        b = np.round(c * E).astype(np.int64)
        b[-1] = E
        return np.maximum.accumulate(b)

    def _issue(self, uh, wh):
        import torch
        if self.direct and uh.is_pinned() and wh.is_pinned() and \
                (uh.data_ptr() | wh.data_ptr()) % 16 == 0:
            return self._issue_direct(uh, wh)
        m = self.mesh
        nq3 = m.nq ** 3
        L = lib()
        D = m.basis.diff
        bounds = self._bounds(m.E)
        main = torch.cuda.current_stream()
        self.s_in.wait_stream(main)
        ev_in, ev_cmp = [], []
        for c in range(self.nchunks):
            a, b = int(bounds[c]) * nq3, int(bounds[c + 1]) * nq3
            with torch.cuda.stream(self.s_in):
                self.ud[a:b].copy_(uh[a:b], non_blocking=True)
                e1 = torch.cuda.Event()
                e1.record(self.s_in)
            self.s_cmp.wait_event(e1)
            e0, ne = int(bounds[c]), int(bounds[c + 1] - bounds[c])
            check(L.nk_bk5(m.N, ne, ptr(D), m.G.data_ptr() + e0 * 6 * nq3 * 8,
                           self.ud.data_ptr() + a * 8, self.wd.data_ptr() + a * 8, 1.0, None,
                           0.0, 1, ne * nq3, None, None, 0, None, None, 0, 0,
                           self.s_cmp.cuda_stream), "bk5")
            e2 = torch.cuda.Event()
            e2.record(self.s_cmp)
            self.s_out.wait_event(e2)
            with torch.cuda.stream(self.s_out):
                wh[a:b].copy_(self.wd[a:b], non_blocking=True)
        main.wait_stream(self.s_out)

    def _issue_stream(self, uh, wh):
        """Direct mode, one kernel: the H2D chunks (and behind each, the
        element count it completes into the device gate) run on the copy
        engine while ONE persistent stage kernel, launched concurrently,
        stages each element's u as soon as its chunk has landed and bulk-
        stores w into the pinned host buffer -- no per-chunk kernel ramp /
        tail gaps in the device -> host write stream."""
        import torch
        m = self.mesh
        nq3 = m.nq ** 3
        L = lib()
        bounds = self._bounds(m.E)
        main = torch.cuda.current_stream()
        self.s_in.wait_stream(main)
        check(L.nk_stream_write_u64(self.gate.data_ptr(), 0, self.s_in.cuda_stream),
              "stream_write_u64")
        with torch.cuda.stream(self.s_in):
            ev0 = torch.cuda.Event()
            ev0.record(self.s_in)
        self.s_cmp.wait_event(ev0)
        with torch.cuda.stream(self.s_in):
            for c in range(self.nchunks):
                a, b = int(bounds[c]) * nq3, int(bounds[c + 1]) * nq3
                self.ud[a:b].copy_(uh[a:b], non_blocking=True)
                # the element count this chunk completes, written by the GPU
                # front end once the copy is done (a tiny H2D copy per chunk
                # measured ~20 us each)
                check(L.nk_stream_write_u64(self.gate.data_ptr(), int(bounds[c + 1]),
                                            self.s_in.cuda_stream), "stream_write_u64")
        old = L.nk_bk5_set_variant(BK5_VARIANTS["stage"])
        L.nk_bk5_set_gate(self.gate.data_ptr())
        try:
            check(L.nk_bk5(m.N, m.E, ptr(m.basis.diff), ptr(m.G), self.ud.data_ptr(),
                           wh.data_ptr(), 1.0, None, 0.0, 1, m.n_local, None, None, 0, None,
                           None, 0, 0, self.s_cmp.cuda_stream), "bk5")
        finally:
            L.nk_bk5_set_gate(None)
            L.nk_bk5_set_variant(old)
        main.wait_stream(self.s_cmp)
        main.wait_stream(self.s_in)

    def _issue_direct(self, uh, wh):
        if self.STREAM:
            return self._issue_stream(uh, wh)
        import torch
        m = self.mesh
        nq3 = m.nq ** 3
        L = lib()
        D = m.basis.diff
        bounds = self._bounds(m.E)
        main = torch.cuda.current_stream()
        self.s_in.wait_stream(main)
        old = L.nk_bk5_set_variant(BK5_VARIANTS["stage"])   # bulk w stores (host memory)
        try:
            for c in range(self.nchunks):
                a, b = int(bounds[c]) * nq3, int(bounds[c + 1]) * nq3
                with torch.cuda.stream(self.s_in):
                    self.ud[a:b].copy_(uh[a:b], non_blocking=True)
                    e1 = torch.cuda.Event()
                    e1.record(self.s_in)
                self.s_cmp.wait_event(e1)
                e0, ne = int(bounds[c]), int(bounds[c + 1] - bounds[c])
                check(L.nk_bk5(m.N, ne, ptr(D), m.G.data_ptr() + e0 * 6 * nq3 * 8,
                               self.ud.data_ptr() + a * 8, wh.data_ptr() + a * 8, 1.0, None,
                               0.0, 1, ne * nq3, None, None, 0, None, None, 0, 0,
                               self.s_cmp.cuda_stream), "bk5")
        finally:
            L.nk_bk5_set_variant(old)
        main.wait_stream(self.s_cmp)


def apply_stiffness_local(u, mesh, basis=None, out=None, elements=None, nchunks=None):
    """Unassembled A_L u_L.  u: (E, nq, nq, nq) or flat,
    CUDA float64 (in place into `out` if given), or a HOST array/tensor
    (numpy or CPU torch, ideally pinned) which is streamed through the device
    in `nchunks` overlapped H2D / BK5 / D2H chunks (a cached CUDA graph for
    pinned buffers) and returned on the host.
    basis defaults to mesh.basis (orders must match)."""
    import torch
    if basis is not None and basis.order != mesh.N:
        raise ContractError(f"contract error: basis order {basis.order} != mesh order {mesh.N}")
    if _is_host(u) and elements is None:
        t = torch.as_tensor(u) if isinstance(u, np.ndarray) else u
        if t.dtype != torch.float64:
            raise ContractError("field must be float64")
        if t.numel() != mesh.n_local:
            raise ContractError(f"contract error: field length {t.numel()} != {mesh.n_local}")
        t = t.contiguous().reshape(-1)
        if out is not None and _is_host(out):
            wh = torch.as_tensor(out).reshape(-1)
        else:
            wh = torch.empty(mesh.n_local, dtype=torch.float64, pin_memory=t.is_pinned())
        if nchunks is None:   # measured best: 8 direct-mode chunks, 6 copy-pipeline chunks
            nchunks = 8 if mesh.N in _HostStream.DIRECT_ORDERS else 6
        hs = getattr(mesh, "_host_stream", None)
        if hs is None or hs.nchunks != nchunks:
            hs = mesh._host_stream = _HostStream(mesh, nchunks)
        hs.run(t, wh)
        torch.cuda.current_stream().synchronize()
        if isinstance(u, np.ndarray):
            return wh.numpy().reshape(np.shape(u))
        return wh.reshape(u.shape)
    t, host = _as_device(u, mesh, 1)
    w = _bk5(t, mesh, 1.0, 0.0, 1, out=out, elements=elements)
    return w.cpu().numpy().reshape(np.shape(u)) if host else w


def apply_helmholtz_local(u, mesh, lam0, lam1, ncomp=1, out=None, elements=None):
    """lam0 * A_L u + lam1 * B u for ncomp (1 or 3) component-major fields."""
    t, host = _as_device(u, mesh, ncomp)
    w = _bk5(t, mesh, lam0, lam1, ncomp, out=out, elements=elements)
    return w.cpu().numpy().reshape(np.shape(u)) if host else w


def apply_mass(u, mesh, out=None):
    """B u: pointwise (nk_pointwise; the BK5 launch with
    lam0 = 0 would stream G needlessly)."""
    import torch
    t, host = _as_device(u, mesh, 1)
    if t.numel() != mesh.n_local:
        raise ContractError(f"contract error: field length {t.numel()} != {mesh.n_local}")
    w = torch.empty_like(t) if out is None else out
    check(lib().nk_pointwise(mesh.n_local, ptr(mesh.B), ptr(t), ptr(w), 1.0, None, stream_ptr()),
          "pointwise")
    return w.cpu().numpy() if host else w


def inner_product(v, u, mesh, comm=None):
    """(v, u)_B = sum_L v B u, deterministic two-stage device reduction
    (SPEC.md:380-388, 554), all-reduced over ranks when comm is given."""
    import torch
    tv, _ = _as_device(v, mesh, 1)
    tu, _ = _as_device(u, mesh, 1)
    n = mesh.n_local
    if tv.numel() != n or tu.numel() != n:
        raise ContractError("contract error: field length mismatch")
    out = torch.zeros(1, dtype=torch.float64, device=mesh.device)
    part = torch.empty(int(lib().nk_cg_partials_len(n)), dtype=torch.float64, device=mesh.device)
    check(lib().nk_wdot(n, ptr(tv), ptr(tu), ptr(mesh.B), ptr(out), ptr(part), stream_ptr()),
          "wdot")
    if comm is not None and comm.size > 1:
        comm.allreduce_sum_(out)
    return float(out.item())


def extract_diagonal(mesh, basis=None, spec="stiffness", gs=None, assemble=True):
    """Jacobi diagonal: closed-form local diag(A_e) on the
    device (nk_local_diag), then gs(+) to assemble.  spec: 'stiffness' or
    ('helmholtz', lam) meaning A + lam*B, or ('helmholtz', lam0, lam1)."""
    import torch
    from .gather_scatter import gs_op, gs_setup
    lam0, lam1 = 1.0, 0.0
    if isinstance(spec, tuple):
        if spec[0] != "helmholtz":
            raise ContractError(f"unknown operator spec {spec!r}")
        lam0, lam1 = (1.0, float(spec[1])) if len(spec) == 2 else (float(spec[1]), float(spec[2]))
    elif spec != "stiffness":
        raise ContractError(f"unknown operator spec {spec!r}")
    D = mesh.basis.device_arrays(mesh.device)[0]
    d = torch.empty((mesh.E, mesh.nq, mesh.nq, mesh.nq), dtype=torch.float64, device=mesh.device)
    check(lib().nk_local_diag(mesh.N, mesh.E, ptr(D), ptr(mesh.G), lam0,
                              ptr(mesh.B) if lam1 else None, lam1, ptr(d), stream_ptr()),
          "local_diag")
    if assemble:
        if gs is None:
            gs = gs_setup(mesh.ids, nq=mesh.nq, device=mesh.device)
        gs_op(gs, d)
    return d


# BK5 variants (nk_bk5_set_variant): declaration order = tie-break order
BK5_VARIANTS = {"kslab": 1, "pencil": 3, "pencil_tma": 4, "pencil2": 5, "seq3": 6, "dmma": 7,
                "stage": 8, "stage2": 9, "pair": 10, "point": 11}
_VARIANT_REPORT = []


def bk5_variant_eligible(name, N, ncomp=1):
    """Which BK5 variants serve an order (the analogue of SPEC.md:426's
    "N_q=12 -> full3d not eligible"): pencil-TMA needs N+1 in {4, 6, 8};
    dmma (FP64 tensor cores, two 8-row tiles) N+1 in 9..16; stage (TMA-staged
    operands) N+1 in 3, 5..16, stage2 N+1 in 9..15, pair N+1 = 16, point N+1 = 3; seq3 serves
    3-component batches only."""
    if name not in BK5_VARIANTS:
        return False
    if name == "pencil_tma":
        return ncomp == 1 and N + 1 in (4, 6, 8)
    if name == "dmma":
        return ncomp == 1 and 9 <= N + 1 <= 16
    if name == "stage":   # TMA-staged u and G in shared memory (bk5_stage.cuh)
        return ncomp == 1 and N + 1 >= 3 and N + 1 != 4
    if name == "stage2":  # stage with two threads per pencil (bk5_stage2.cuh)
        return ncomp == 1 and 9 <= N + 1 <= 15
    if name == "pair":    # one element per CTA pair (cluster; bk5_pair.cuh)
        return ncomp == 1 and N + 1 == 16
    if name == "point":   # one thread per point (bk5_point.cuh)
        return ncomp == 1 and N + 1 == 3
    if name == "seq3":   # 3 components back to back per CTA (bk5_pencil NC = 3)
        return ncomp == 3
    return True


def select_kernel_variant(mesh, candidates=None, reps=20, force=None, ncomp=1):
    """Measured BK5 variant choice on `mesh` (the runtime
    analogue of the paper's "2D or 3D thread structure ... whichever is more
    performant"): every eligible candidate runs `reps`
    timed applies (CUDA events, after one warm-up); the lowest median wins,
    ties broken by declaration order; `force` (a variant name) skips the
    benchmark.  The choice is installed process-wide (nk_bk5_set_variant) and
    recorded in variant_report().  Returns the chosen name."""
    import statistics

    import torch
    names = list(BK5_VARIANTS) if candidates is None else list(candidates)
    for nme in names:
        if nme not in BK5_VARIANTS:
            raise ContractError(f"unknown BK5 variant {nme!r} (built: {list(BK5_VARIANTS)})")
    if force is not None:
        if force not in BK5_VARIANTS:
            raise ContractError(f"unknown BK5 variant {force!r}")
        lib().nk_bk5_set_variant(BK5_VARIANTS[force])
        _VARIANT_REPORT.append({"N": mesh.N, "E": mesh.E, "chosen": force, "forced": True})
        return force
    elig = [n for n in names if bk5_variant_eligible(n, mesh.N, ncomp)]
    if not elig:
        raise ContractError("no eligible BK5 variant among the candidates")
    u = torch.randn(mesh.n_local * ncomp, dtype=torch.float64, device=mesh.device)
    w = torch.empty_like(u)
    old = lib().nk_bk5_set_variant(0)
    times = {}
    try:
        for nme in elig:
            lib().nk_bk5_set_variant(BK5_VARIANTS[nme])
            _bk5(u, mesh, 1.0, 0.0, ncomp, out=w)
            ts = []
            for _ in range(max(1, int(reps))):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                _bk5(u, mesh, 1.0, 0.0, ncomp, out=w)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            times[nme] = statistics.median(ts)
    finally:
        lib().nk_bk5_set_variant(old)
    best = min(elig, key=lambda n: (times[n], elig.index(n)))
    lib().nk_bk5_set_variant(BK5_VARIANTS[best])
    _VARIANT_REPORT.append({"N": mesh.N, "E": mesh.E, "chosen": best, "forced": False,
                            "median_ms": {k: round(v, 5) for k, v in times.items()}})
    return best


def reset_kernel_variant():
    """Back to the measured per-order table (nk_bk5_set_variant(0))."""
    lib().nk_bk5_set_variant(0)


def variant_report():
    """Selections made by select_kernel_variant (the timing report entry of
    SPEC.md:425)."""
    return list(_VARIANT_REPORT)
