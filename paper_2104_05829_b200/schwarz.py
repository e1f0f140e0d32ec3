"""Overlapping Schwarz smoothers with FDM local solves.

Drop-in for nekmini's ``fdm_local_solve`` and ``schwarz_smooth`` (SPEC.md:
410-418, 499-507) and the smoother kinds asm / ras / cheby_asm / cheby_ras of
``SmootherConfig``:
each spectral element is extended by one layer of points from its face
neighbours ((N+3)^3 boxes), the residual there is solved exactly for an
axis-aligned box surrogate by fast diagonalisation, and the results are
combined by exchange-and-add with the counting weight (ASM) or kept per
element (RAS).

Per application (all libnekb200 launches on the current stream, CUDA-graph
capturable, skipped once the PCG state says done):
  [multi-rank]      nk_gather_diff packs r (- A e) at the face-inward layers
                    neighbour ranks need; one pairwise exchange;
  nk_fdm            gather r (- A e) on the extended boxes, 6 tensor
                    contractions + inverse spectrum, write the extended (ASM)
                    or own-point (RAS) solution;
  gs                ASM: the extended-id gs handle (SPEC.md:504's "dedicated gs
                    handle"); RAS: the operator's own QQ^T;
  nk_schwarz_post   z = mask * weight * (own points), fused with the
                    Chebyshev update d = a d + b z, e (+)= d.
Setup (face-neighbour map from global ids, element lengths, the batched 1-D
generalised eigenproblems, extended ids and counting weights) runs once on the
host/device.  oracle/schwarz.py states the same algorithm on the CPU.
"""

import numpy as np

from ._lib import ContractError, check, lib, ptr, stream_ptr

__all__ = ["SchwarzSmoother", "fdm_local_solve", "schwarz_smooth", "face_source_map",
           "fdm_1d_batch", "KINDS"]

KINDS = ("asm", "ras")
_NBR, _NEU, _DIR = 0, 1, 2
_FACE_AXES = ((0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1))


def _face_slice(nq, axis, side, inward=False):
    p = (1 if side == 0 else nq - 2) if inward else (0 if side == 0 else nq - 1)
    s = [slice(None)] * 4
    s[3 - axis] = p
    return tuple(s)


def _face_pairs(srt):
    """Rows of srt (sorted face id sets) that are equal, as index pairs.
    Groups by a 64-bit polynomial hash of the row (fast), then verifies the
    candidate pairs exactly; any collision or a group of more than two falls
    back to the exact (slow) row-unique path."""
    with np.errstate(over="ignore"):
        key = np.zeros(len(srt), dtype=np.uint64)
        for q in range(srt.shape[1]):
            key = key * np.uint64(0x9E3779B97F4A7C15) + srt[:, q].astype(np.uint64)
    order = np.argsort(key, kind="stable")
    k = key[order]
    same = k[1:] == k[:-1]
    triple = same[1:] & same[:-1]
    r0, r1 = order[:-1][same], order[1:][same]
    if not triple.any() and np.array_equal(srt[r0], srt[r1]):
        return r0, r1
    _, grp, cnt = np.unique(srt, axis=0, return_inverse=True, return_counts=True)
    if np.any(cnt > 2):
        raise ContractError("a face id set is held by more than two element faces")
    grp = grp.ravel()
    order = np.argsort(grp, kind="stable")
    g = grp[order]
    same = g[1:] == g[:-1]
    return order[:-1][same], order[1:][same]


def face_source_map(ids, E, N):
    """fmap[e, f, a, b]: local index of the point one layer inside the face
    neighbour across face f (x- x+ y- y+ z- z+) at e's face point (a, b)
    (tangential slow, fast); -1 without a neighbour.  Neighbours are the
    faces holding the same (N+1)^2 global ids (HEXMESH and periodic meshes
    work unchanged).  Vectorised host setup; int64 (E, 6, nq, nq)."""
    nq = N + 1
    ids = np.asarray(ids, dtype=np.int64).reshape(E, nq, nq, nq)
    loc = np.arange(E * nq ** 3, dtype=np.int64).reshape(E, nq, nq, nq)
    fid = np.stack([ids[_face_slice(nq, a, s)].reshape(E, nq * nq) for a, s in _FACE_AXES], 1)
    finw = np.stack([loc[_face_slice(nq, a, s, True)].reshape(E, nq * nq)
                     for a, s in _FACE_AXES], 1)
    fid = fid.reshape(E * 6, nq * nq)
    finw = finw.reshape(E * 6, nq * nq)
    fmap = np.full((E * 6, nq * nq), -1, dtype=np.int64)
    if E == 0:
        return fmap.reshape(E, 6, nq, nq)
    srt = np.sort(fid, axis=1)
    r0, r1 = _face_pairs(srt)
    A = np.concatenate([r0, r1])
    B = np.concatenate([r1, r0])
    if len(A):
        ob = np.argsort(fid[B], axis=1, kind="stable")
        oa = np.argsort(fid[A], axis=1, kind="stable")
        rank = np.empty_like(oa)
        np.put_along_axis(rank, oa, np.arange(nq * nq)[None, :].repeat(len(A), 0), axis=1)
        pos = np.take_along_axis(ob, rank, axis=1)
        fmap[A] = np.take_along_axis(finw[B], pos, axis=1)
    return fmap.reshape(E, 6, nq, nq)


def fdm_1d_batch(D, w, h, left, right, device="cpu"):
    """Batched extended 1-D generalised eigenproblems (oracle/schwarz.py:
    fdm_1d): h (B,), left/right (B,) side kinds 0 nbr / 1 neu / 2 dir.
    Returns float64 torch tensors on `device`: S (B, N+3, N+3) with
    S^T M S = I and lam (B, N+3), +inf on the modes of dropped points
    (decoupled with a -1 diagonal, so eigh isolates them).  The restricted
    matrices are built directly (own element on points 1..N+1, the left /
    right neighbour's two points next to the shared face when present) and
    solved by batched eigh on the device (cuSOLVER on a GPU)."""
    import torch
    f64 = torch.float64
    def _t(x, dt=f64):
        if isinstance(x, torch.Tensor):
            return x.to(device=device, dtype=dt)
        return torch.as_tensor(np.array(x), device=device, dtype=dt)
    D, w, h = _t(D), _t(w), _t(h)
    left, right = _t(left, torch.int64), _t(right, torch.int64)
    N = w.numel() - 1
    nb = h.numel()
    K1 = D.T @ (w[:, None] * D)
    g = (2.0 / h)[:, None, None]
    K = torch.zeros((nb, N + 3, N + 3), dtype=f64, device=device)
    M = torch.zeros((nb, N + 3), dtype=f64, device=device)
    K[:, 1:N + 2, 1:N + 2] = g * K1
    M[:, 1:N + 2] = (h / 2.0)[:, None] * w
    ln = (left == _NBR).to(f64)
    rn = (right == _NBR).to(f64)
    # left neighbour: its local points N-1, N -> restricted 0, 1
    K[:, 0:2, 0:2] += (ln[:, None, None] * g) * K1[N - 1:N + 1, N - 1:N + 1]
    M[:, 0:2] += (ln * h / 2.0)[:, None] * w[N - 1:N + 1]
    # right neighbour: its local points 0, 1 -> restricted N+1, N+2
    K[:, N + 1:N + 3, N + 1:N + 3] += (rn[:, None, None] * g) * K1[0:2, 0:2]
    M[:, N + 1:N + 3] += (rn * h / 2.0)[:, None] * w[0:2]
    keep = torch.ones((nb, N + 3), dtype=torch.bool, device=device)
    keep[:, 0] = left == _NBR
    keep[:, 1] = left != _DIR
    keep[:, N + 2] = right == _NBR
    keep[:, N + 1] = right != _DIR
    drop = ~keep
    K = torch.where(drop[:, :, None] | drop[:, None, :], torch.zeros((), dtype=f64, device=device), K)
    idx = torch.arange(N + 3, device=device)
    K[:, idx, idx] = torch.where(drop, torch.full((), -1.0, dtype=f64, device=device),
                                 K[:, idx, idx])
    M = torch.where(drop, torch.ones((), dtype=f64, device=device), M)
    Mh = 1.0 / torch.sqrt(M)
    Ks = Mh[:, :, None] * K * Mh[:, None, :]
    lam = torch.empty((nb, N + 3), dtype=f64, device=device)
    V = torch.empty_like(Ks)
    CH = 1 << 14          # cuSOLVER batched syev rejects batches >= 32768
    for c0 in range(0, nb, CH):
        lam[c0:c0 + CH], V[c0:c0 + CH] = torch.linalg.eigh(Ks[c0:c0 + CH])
    S = Mh[:, :, None] * V
    lam = torch.where(lam < -0.5, torch.full((), float("inf"), dtype=f64, device=device), lam)
    return S, lam


def _face_hashes(srt):
    """Two independent 64-bit polynomial hashes of sorted face id rows."""
    with np.errstate(over="ignore"):
        k1 = np.zeros(len(srt), dtype=np.uint64)
        k2 = np.zeros(len(srt), dtype=np.uint64)
        for q in range(srt.shape[1]):
            v = srt[:, q].astype(np.uint64)
            k1 = k1 * np.uint64(0x9E3779B97F4A7C15) + v
            k2 = k2 * np.uint64(0xC2B2AE3D27D4EB4F) + (v ^ np.uint64(0x5851F42D4C957F2D))
    return k1.view(np.int64), k2.view(np.int64)


def remote_face_plan(ids, fmap, E, N, comm):
    """Cross-rank face neighbours of the extended boxes (collective).

    Faces without a local neighbour are matched across ranks by their global
    id sets (two 64-bit hashes; owner rank = hash mod P, like the gs halo
    discovery).  For every matched face both ranks list the face points in
    the same order -- (face hashes, face point global id) -- so rank p's
    i-th received value is the neighbour's point one layer inside the face at
    p's i-th listed face point.  Returns (fmap with entries -(2 + slot) for
    remote sources, {peer: local indices to send}, {peer: receive count},
    total receive count)."""
    nq = N + 1
    P, rank = comm.size, comm.rank
    ids = np.asarray(ids, dtype=np.int64).reshape(E, nq, nq, nq)
    loc = np.arange(E * nq ** 3, dtype=np.int64).reshape(E, nq, nq, nq)
    fmap = fmap.copy()
    cand = np.argwhere(fmap[:, :, 0, 0] == -1)                      # (e, f)
    rows_g, rows_in = [], []
    for e, f in cand:
        axis, side = _FACE_AXES[f]
        rows_g.append(ids[e][_face_slice(nq, axis, side)[1:]].reshape(-1))
        rows_in.append(loc[e][_face_slice(nq, axis, side, True)[1:]].reshape(-1))
    nc = len(cand)
    G = np.array(rows_g, dtype=np.int64).reshape(nc, nq * nq)
    IN = np.array(rows_in, dtype=np.int64).reshape(nc, nq * nq)
    k1, k2 = _face_hashes(np.sort(G, axis=1)) if nc else (np.zeros(0, np.int64),) * 2
    owner = (k1.view(np.uint64) % np.uint64(P)).astype(np.int64)
    parts = [np.stack([k1[owner == q], k2[owner == q], np.flatnonzero(owner == q)], 1).ravel()
             for q in range(P)]
    got = comm.alltoallv_int64(parts)
    # owner side: pair equal keys held by two different ranks
    recs = [(int(a), int(b), src, int(c)) for src in range(P)
            for a, b, c in got[src].reshape(-1, 3)]
    recs.sort()
    replies = [[] for _ in range(P)]
    i = 0
    while i < len(recs):
        j = i
        while j < len(recs) and recs[j][:2] == recs[i][:2]:
            j += 1
        grp = recs[i:j]
        if len(grp) == 2 and grp[0][2] != grp[1][2]:
            (_, _, ra, ca), (_, _, rb, cb) = grp
            replies[ra] += [ca, rb]
            replies[rb] += [cb, ra]
        elif len(grp) > 2:
            raise ContractError("a face id set is held by more than two element faces")
        i = j
    back = comm.alltoallv_int64([np.array(r, dtype=np.int64) for r in replies])
    matched = np.concatenate([b.reshape(-1, 2) for b in back]) if P else np.zeros((0, 2))
    send_idx, recv_cnt, entries = {}, {}, {}
    for c, peer in matched:
        e, f = cand[c]
        for a_b in range(nq * nq):
            entries.setdefault(int(peer), []).append(
                (int(k1[c]), int(k2[c]), int(G[c, a_b]), int(IN[c, a_b]), int(e), int(f), a_b))
    off = 0
    for peer in sorted(entries):
        lst = sorted(entries[peer])
        send_idx[peer] = np.array([t[3] for t in lst], dtype=np.int64)
        recv_cnt[peer] = len(lst)
        for slot, t in enumerate(lst):
            e, f, a_b = t[4], t[5], t[6]
            fmap[e, f, a_b // nq, a_b % nq] = -(2 + off + slot)
        off += len(lst)
    return fmap, send_idx, recv_cnt, off


class SchwarzSmoother:
    """z = S r for a PoissonOperator: kind 'asm' or 'ras'.  Across ranks the
    face-inward layers of neighbour ranks are exchanged before each solve, and
    ASM's extended gs runs over the ranks (the remote sources' global ids are
    exchanged once at setup);
    precision 64, or 32 (local solves in FP32, fields FP64 -- the paper's
    32-bit smoothing, SmootherConfig.precision SPEC.md:463).

    Buffers are preallocated; ``apply`` writes into caller buffers so the
    smoother can sit inside a captured CUDA graph (MultigridHierarchy)."""

    def __init__(self, op, kind="asm", precision=64):
        import torch
        from .gather_scatter import gs_setup
        from .mesh import mesh_coordinates
        if kind not in KINDS:
            raise ContractError(f"unknown Schwarz kind {kind!r} (built: {KINDS})")
        if op.ncomp != 1:
            raise ContractError("Schwarz smoothing is built for scalar operators")
        if precision not in (32, 64):
            raise ContractError(f"precision must be 32 or 64, got {precision!r}")
        self.precision = int(precision)
        comm = op.gs.comm
        self.comm = comm if (comm is not None and comm.size > 1) else None
        m = op.mesh
        self.op, self.kind, self.mesh = op, kind, m
        N, E, nq = m.N, m.E, m.nq
        nqe = N + 3
        self.N, self.E, self.nqe = N, E, nqe
        dev = m.device
        ids = m.ids.detach().cpu().numpy().astype(np.int64).ravel()
        mask = m.mask.detach().cpu().numpy().reshape(E, nq, nq, nq)
        fmap = face_source_map(ids, E, N)
        self.send_idx, self.recv_cnt = {}, {}
        if self.comm is not None:
            # faces whose neighbour lives on another rank read that rank's
            # inward layer from a receive buffer (one exchange per smoothing)
            fmap, sidx, self.recv_cnt, nrecv = remote_face_plan(ids, fmap, E, N, self.comm)
            self.send_idx = {q: torch.as_tensor(v.astype(np.int32), device=dev)
                             for q, v in sidx.items()}
            self.send_buf = {q: torch.zeros(len(v), dtype=torch.float64, device=dev)
                             for q, v in sidx.items()}
            self.rx = torch.zeros(max(nrecv, 1), dtype=torch.float64, device=dev)
            self.recv_slices = {}
            o = 0
            for q in sorted(self.recv_cnt):
                self.recv_slices[q] = self.rx[o:o + self.recv_cnt[q]]
                o += self.recv_cnt[q]
            # the global ids of the remote sources (ASM's extended numbering)
            xdev = dev if self.comm.backend == "nccl" else "cpu"
            rid = torch.zeros(max(nrecv, 1), dtype=torch.int64, device=xdev)
            sid = {q: torch.as_tensor(ids[v], device=xdev) for q, v in sidx.items()}
            ridv, o = {}, 0
            for q in sorted(self.recv_cnt):
                ridv[q] = rid[o:o + self.recv_cnt[q]]
                o += self.recv_cnt[q]
            self.comm.exchange(sid, ridv)
            rid = rid.cpu()
            self.remote_ids = rid.numpy()[:nrecv]
        # side kinds
        kinds = np.empty((E, 6), dtype=np.int64)
        for f, (axis, side) in enumerate(_FACE_AXES):
            masked = np.all(mask[_face_slice(nq, axis, side)].reshape(E, -1) == 0, axis=1)
            kinds[:, f] = np.where(fmap[:, f, 0, 0] != -1, _NBR, np.where(masked, _DIR, _NEU))
        self.kinds = kinds
        # element lengths (mean distance between opposite faces)
        X = mesh_coordinates(m)
        h = torch.zeros((E, 3), dtype=torch.float64, device=dev)
        for d in range(3):
            lo, hi = _face_slice(nq, d, 0), _face_slice(nq, d, 1)
            diff = torch.stack([X[c][hi] - X[c][lo] for c in range(3)])
            h[:, d] = torch.sqrt((diff ** 2).sum(0)).reshape(E, -1).mean(1)
        self.h = h
        b = m.basis
        S, lam = fdm_1d_batch(b.diff, b.weights, h.reshape(-1), kinds[:, 0::2].reshape(-1),
                              kinds[:, 1::2].reshape(-1), device=dev)
        S = S.reshape(E, 3, nqe, nqe)
        lam = lam.reshape(E, 3, nqe)
        lam1 = float(op.lam1)
        if lam1 == 0.0:
            neu = torch.as_tensor(np.all(kinds == _NEU, axis=1), device=dev)
            if bool(neu.any()):   # pure-Neumann surrogate: shift by eps = 1e-8 max(Lambda)
                ln_ = lam[neu]
                fin = torch.isfinite(ln_)
                eps = 1e-8 * torch.where(fin, ln_, torch.zeros_like(ln_)).amax(dim=2).sum(dim=1)
                lam[neu] = torch.where(fin, ln_ + eps[:, None, None] / 3.0, ln_)
        self.S = S.contiguous()
        self.lam = lam.contiguous()
        if self.precision == 32:      # local solves in FP32 (+inf stays +inf)
            self.S = self.S.float().contiguous()
            self.lam = self.lam.float().contiguous()
        self.fmap = torch.as_tensor(fmap.astype(np.int32), device=dev).contiguous()
        self.mask = m.mask.reshape(-1)
        n = E * nq ** 3
        self.n = n
        if kind == "asm":
            src = np.full((E, nqe, nqe, nqe), -1, dtype=np.int64)
            src[:, 1:nq + 1, 1:nq + 1, 1:nq + 1] = np.arange(n).reshape(E, nq, nq, nq)
            for fi, (axis, side) in enumerate(_FACE_AXES):
                s = [slice(None), slice(1, nq + 1), slice(1, nq + 1), slice(1, nq + 1)]
                s[3 - axis] = 0 if side == 0 else nqe - 1
                src[tuple(s)] = fmap[:, fi]
            src = src.reshape(-1)
            ext_ids = np.where(src >= 0, ids[np.maximum(src, 0)], 0)
            if self.comm is not None:      # remote sources carry the neighbour's ids
                rem = src <= -2
                ext_ids[rem] = self.remote_ids[-src[rem] - 2]
            self.ext_gs = gs_setup(ext_ids, comm=self.comm, device=dev)
            self.buf = torch.zeros(E * nqe ** 3, dtype=torch.float64, device=dev)
            cnt = torch.as_tensor((src != -1).astype(np.float64), device=dev)
            self._gs(self.ext_gs, cnt)
            own = cnt.view(E, nqe, nqe, nqe)[:, 1:nq + 1, 1:nq + 1, 1:nq + 1].reshape(-1)
            self.W = (1.0 / own).contiguous()
            self.ext_ids = ext_ids
        else:
            self.ext_gs = None
            self.buf = torch.zeros(n, dtype=torch.float64, device=dev)
            self.W = op.weights

    @staticmethod
    def _gs(h, w, st=None):
        from .gather_scatter import _halo_exchange, _halo_finish, _halo_start, _local
        if h.comm is None or h.comm.size == 1:
            _local(h, w, "+", 1, st=st)
            return
        _halo_start(h, w, st=st)
        _halo_exchange(h)
        _local(h, w, "+", 1, st=st, part=h.seg_rest)
        _halo_finish(h, w, "+", st=st)

    @property
    def launches(self):
        return 3

    def fdm(self, r, out, sub=None, res_out=None, out_ext=True, st=None):
        """FDM local solves of the extended residual of r - sub (nk_fdm, or
        nk_fdm32 in the 32-bit smoothing mode)."""
        fn = lib().nk_fdm32 if self.precision == 32 else lib().nk_fdm
        rx = None
        if self.comm is not None:
            L, s = lib(), stream_ptr()
            for q, idx in self.send_idx.items():
                check(L.nk_gather_diff(idx.numel(), ptr(idx), ptr(r), ptr(sub),
                                       ptr(self.send_buf[q]), ptr(st), s), "gather_diff")
            self.comm.exchange(self.send_buf, self.recv_slices)
            rx = self.rx
        check(fn(self.N, self.E, ptr(r), ptr(sub), ptr(rx), ptr(res_out), ptr(self.fmap),
                           ptr(self.S), ptr(self.lam), float(self.op.lam0), float(self.op.lam1),
                           ptr(out), int(out_ext), ptr(st), stream_ptr()), "fdm")

    def apply(self, r, e, sub=None, res_out=None, d=None, a=0.0, b=1.0, e_acc=False, st=None):
        """z = S (r - sub); d = a d + b z (d optional); e = [e +] d.
        res_out receives r - sub (must not alias r or sub)."""
        asm = self.kind == "asm"
        self.fdm(r, self.buf, sub, res_out, out_ext=asm, st=st)
        self._gs(self.ext_gs if asm else self.op.gs, self.buf, st)
        check(lib().nk_schwarz_post(self.N, self.E, ptr(self.buf), int(asm), ptr(self.W),
                                    ptr(self.mask), ptr(d), ptr(e), float(a), float(b),
                                    int(bool(e_acc)), ptr(st), stream_ptr()), "schwarz_post")
        return e

    def __call__(self, r):
        import torch
        rf = r.reshape(-1).contiguous()
        if rf.numel() != self.n:
            raise ContractError(f"contract error: field length {rf.numel()} != {self.n}")
        z = torch.empty_like(rf)
        self.apply(rf, z)
        return z.view_as(r)


def fdm_local_solve(smoother, residual):
    """Extended FDM solution u_ext [E][(N+3)^3] of an assembled residual
    (SPEC.md:410-418), a new tensor."""
    import torch
    rf = residual.reshape(-1).contiguous()
    if rf.numel() != smoother.n:
        raise ContractError(f"contract error: field length {rf.numel()} != {smoother.n}")
    out = torch.empty(smoother.E * smoother.nqe ** 3, dtype=torch.float64, device=rf.device)
    smoother.fdm(rf, out, out_ext=True)
    return out.view(smoother.E, smoother.nqe, smoother.nqe, smoother.nqe)


def schwarz_smooth(smoother, r):
    """z = S r; a new tensor."""
    return smoother(r)
