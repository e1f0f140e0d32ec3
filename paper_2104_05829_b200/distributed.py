"""Ranks, id discovery and the pairwise halo exchange (
PAPER.md:92-141).

One process per GPU.  ``RankComm`` wraps a torch.distributed process group
(NCCL over NVLink/NVSwitch on the GPU box; gloo for the CPU tests).  The
SPEC's three strategies collapse to one on an NVSwitch node: every peer is at
full bandwidth, ngh <= 7 for an RCB box partition at P = 8, so the pairwise
exchange is always chosen.

Host plan construction (``build_halo_plan``), all collective and
deterministic:
  1. candidates = this rank's ids that sit on element faces (element-interior
     GLL points are never shared in a conforming mesh);
  2. each candidate id g is sent to its owner rank g % P (all-to-all);
  3. the owner reports back, for every id held by >= 2 ranks, the bitmask of
     holder ranks (all-to-all);
  4. halo ids H = ids with >= 2 holders, sorted ascending; per neighbour q the
     send/recv order is H restricted to ids q also holds -- both sides derive
     the same order without further messages.
The exchange carries every local copy of a halo id (not a pre-summed
partial): the combine then folds all contributions of an id in ascending
(rank, local index) order -- exactly the canonical order of SPEC.md:205 -- so
multi-rank results are bit-identical to the single-process fold and to every
other rank's copy.  Local segments of halo ids are therefore not
folded locally; only ids private to the rank use the local plan.
"""

import numpy as np


class RankComm:
    """Collective context for one rank.

    group: a torch.distributed ProcessGroup (None = default group).
    staging: 'device' exchanges device buffers directly (NCCL); 'host' stages
    them through host memory (the paper's host-staged variant; used with gloo
    when several ranks share one GPU in tests)."""

    def __init__(self, group=None, staging=None, transport="auto"):
        """transport: 'ipc' -- halo values pushed by kernels straight into the
        neighbours' receive buffers over NVLink peer memory (CUDA IPC);
        'p2p' -- torch.distributed send/recv (NCCL or gloo); 'auto' -- 'ipc'
        when every neighbour's buffer can be mapped, else 'p2p'."""
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.backend = backend
        self.staging = staging or ("device" if backend == "nccl" else "host")
        if transport not in ("auto", "ipc", "p2p"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport

    # ------------------------------------------------------------ helpers
    def alltoallv_int64(self, parts):
        """parts: list of P int64 numpy arrays (one per destination).
        Returns the list of P arrays received (one per source)."""
        import torch
        dist = self.dist
        P = self.size
        dev = "cuda" if self.backend == "nccl" else "cpu"
        send_counts = torch.tensor([len(p) for p in parts], dtype=torch.int64, device=dev)
        recv_counts = torch.empty(P, dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc = [int(v) for v in send_counts.cpu()]
        rc = [int(v) for v in recv_counts.cpu()]
        send = torch.as_tensor(np.concatenate(parts).astype(np.int64) if sum(sc) else
                               np.zeros(0, np.int64), device=dev)
        recv = torch.empty(sum(rc), dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv, send, rc, sc, group=self.group)
        r = recv.cpu().numpy()
        offs = np.r_[0, np.cumsum(rc)]
        return [r[offs[q]:offs[q + 1]] for q in range(P)]

    def enable_board(self, device="cuda"):
        """Map every rank's scalar board (collective).  Afterwards
        allreduce_sum_ on <= 4 CUDA doubles runs as nk_board_allreduce
        (peer-memory, deterministic, graph-capturable).  Returns success."""
        if getattr(self, "board", None) is not None:
            return True
        if self.transport == "p2p" or self.size > 8:
            return False
        try:
            self.board = IpcBoard(self, device)   # raises on every rank or none
        except Exception:
            if self.transport == "ipc":
                raise
            self.board = None
        return self.board is not None

    def allreduce_sum_(self, t):
        b = getattr(self, "board", None)
        if b is not None and t.is_cuda and t.numel() <= 4 and t.dtype.itemsize == 8:
            b.allreduce_(t)
            return t
        if self.staging == "host" and t.is_cuda:
            h = t.detach().cpu()
            self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
            return t
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def barrier(self):
        self.dist.barrier(group=self.group)

    def exchange_bytes(self, sends):
        """{peer: bytes} -> {peer: bytes} of equal length (setup metadata)."""
        import torch
        if not sends:
            return {}
        dev = "cuda" if self.backend == "nccl" else "cpu"
        st = {q: torch.tensor(list(b), dtype=torch.uint8, device=dev) for q, b in sends.items()}
        rv = {q: torch.zeros(len(b), dtype=torch.uint8, device=dev) for q, b in sends.items()}
        self.exchange(st, rv)
        return {q: bytes(t.cpu().numpy().tolist()) for q, t in rv.items()}

    def exchange(self, sends, recvs):
        """Pairwise exchange: sends/recvs are {peer: tensor}.  Blocking on the
        current stream (NCCL enqueues on it)."""
        dist = self.dist
        if not sends and not recvs:
            return
        if self.staging == "host":
            import torch
            hs = {q: t.detach().to("cpu") for q, t in sends.items()}
            hr = {q: torch.empty(t.shape, dtype=t.dtype) for q, t in recvs.items()}
            ops = [dist.P2POp(dist.isend, hs[q], q, self.group) for q in sorted(hs)]
            ops += [dist.P2POp(dist.irecv, hr[q], q, self.group) for q in sorted(hr)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for q, t in recvs.items():
                t.copy_(hr[q])
            return
        ops = [dist.P2POp(dist.isend, sends[q], q, self.group) for q in sorted(sends)]
        ops += [dist.P2POp(dist.irecv, recvs[q], q, self.group) for q in sorted(recvs)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()


class HaloPlan:
    """Host-side arrays describing the cross-rank part of QQ^T for one rank.

    hids        sorted halo ids (held by >= 2 ranks)
    masks       holder-rank bitmask per halo id
    neighbors   sorted neighbour ranks; ngh = len(neighbors)
    dst_start/dst_idx   CSR: all local copies of each halo id (ascending); the
                        own contributions are buf[0:len(dst_idx)] = w[dst_idx]
    send_idx[q] local indices sent to q: copies of the ids shared with q, ids
                ascending, copies ascending
    recv_off[q], recv_len[q]   where q's contributions land in buf
    src_start/src_idx   CSR into buf: the contributions of each halo id in
                        ascending (rank, local index) order
    """


def _face_point_mask(nq):
    r = np.arange(nq)
    on = (r == 0) | (r == nq - 1)
    return (on[:, None, None] | on[None, :, None] | on[None, None, :]).ravel()


def build_halo_plan(ids, comm, nq=None):
    """Collective discovery of rank-shared ids (see module doc)."""
    import torch
    ids = np.asarray(ids, dtype=np.int64).ravel()
    P, me = comm.size, comm.rank
    if P > 62:
        raise ValueError("holder bitmasks support at most 62 ranks")
    if nq is not None:
        fm = np.tile(_face_point_mask(nq), len(ids) // nq ** 3)
        cand = np.unique(ids[fm & (ids > 0)])
    else:
        cand = np.unique(ids[ids > 0])
    owner = cand % P
    got = comm.alltoallv_int64([cand[owner == q] for q in range(P)])
    # owner side: (id, holder-rank) pairs -> bitmask per id held by >= 2 ranks
    gid = np.concatenate(got) if got else np.zeros(0, np.int64)
    src = np.concatenate([np.full(len(g), q, dtype=np.int64) for q, g in enumerate(got)])
    replies = [np.zeros(0, np.int64)] * P
    if len(gid):
        o = np.lexsort((src, gid))
        gid, src = gid[o], src[o]
        u, cnt = np.unique(gid, return_counts=True)
        bits = np.zeros(len(u), dtype=np.int64)
        np.bitwise_or.at(bits, np.repeat(np.arange(len(u)), cnt), np.left_shift(1, src))
        shared = cnt >= 2
        us, bs = u[shared], bits[shared]
        replies = []
        for q in range(P):
            sel = (bs >> q) & 1 == 1
            replies.append(np.stack([us[sel], bs[sel]], axis=1).ravel())
    back = comm.alltoallv_int64(replies)
    rec = np.concatenate([b.reshape(-1, 2) for b in back]) if back else np.zeros((0, 2), np.int64)
    rec = rec[np.argsort(rec[:, 0], kind="stable")] if len(rec) else rec.reshape(0, 2)
    plan = HaloPlan()
    plan.rank, plan.size = me, P
    plan.hids = rec[:, 0].copy()
    masks = rec[:, 1].copy()
    nh = len(plan.hids)
    plan.masks = masks
    bitsP = ((masks[:, None] >> np.arange(P, dtype=np.int64)[None, :]) & 1).astype(bool)
    nb = [q for q in range(P) if q != me and bool(bitsP[:, q].any())]
    plan.neighbors, plan.ngh = nb, len(nb)
    # local copies of every halo id (ascending local index)
    order = np.argsort(ids, kind="stable")
    sids = ids[order]
    lo = np.searchsorted(sids, plan.hids, side="left")
    hi = np.searchsorted(sids, plan.hids, side="right")
    if np.any(hi <= lo):
        raise RuntimeError("halo id without a local copy (inconsistent discovery)")
    mult = hi - lo
    plan.dst_start = np.r_[0, np.cumsum(mult)].astype(np.int64)
    plan.dst_idx = order[_ranges(lo, mult)] if nh else np.zeros(0, np.int64)
    plan.rep = order[lo] if nh else np.zeros(0, np.int64)
    own_len = len(plan.dst_idx)
    # ids shared with each neighbour (positions into hids, ascending id)
    shared_pos = {q: np.flatnonzero(bitsP[:, q]).astype(np.int64) for q in nb}
    plan.send_idx = {q: plan.dst_idx[_ranges(plan.dst_start[shared_pos[q]], mult[shared_pos[q]])]
                     for q in nb}
    # setup exchange: how many copies each neighbour holds of each shared id
    sends = {q: torch.as_tensor(mult[shared_pos[q]].astype(np.int64)) for q in nb}
    recvs = {q: torch.zeros(len(shared_pos[q]), dtype=torch.int64) for q in nb}
    if comm.backend == "nccl":
        sends = {q: t.cuda() for q, t in sends.items()}
        recvs = {q: t.cuda() for q, t in recvs.items()}
    comm.exchange(sends, recvs)
    their = {q: recvs[q].cpu().numpy().astype(np.int64) for q in nb}
    plan.recv_off, plan.recv_len, off = {}, {}, own_len
    for q in nb:
        plan.recv_off[q] = off
        plan.recv_len[q] = int(their[q].sum())
        off += plan.recv_len[q]
    plan.buf_len = off
    # contributions of halo id t from rank q: cnt[t, q] values starting at
    # buf[start[t, q]]; the combine reads them row by row (t ascending), ranks
    # ascending within a row -- the canonical (rank, local index) order
    cnt = np.zeros((nh, P), dtype=np.int64)
    start = np.zeros((nh, P), dtype=np.int64)
    cnt[:, me] = mult
    start[:, me] = plan.dst_start[:-1]
    for q in nb:
        sp = shared_pos[q]
        cnt[sp, q] = their[q]
        start[sp, q] = plan.recv_off[q] + np.r_[0, np.cumsum(their[q])[:-1]]
    plan.src_start = np.r_[0, np.cumsum(cnt.sum(axis=1))].astype(np.int64)
    plan.src_idx = _ranges(start.ravel(), cnt.ravel())
    return plan


def _ranges(starts, counts):
    """Concatenation of arange(s, s + c) for (s, c) pairs, vectorised."""
    starts = np.asarray(starts, dtype=np.int64)
    counts = np.asarray(counts, dtype=np.int64)
    if len(counts) == 0 or counts.sum() == 0:
        return np.zeros(0, np.int64)
    tot = int(counts.sum())
    offs = np.repeat(np.cumsum(counts) - counts, counts)
    return np.repeat(starts, counts) + (np.arange(tot) - offs)


def boundary_elements(plan, n_elem, nq3):
    """Elements holding at least one halo id (evaluated first)."""
    flag = np.zeros(n_elem, dtype=bool)
    if len(plan.dst_idx):
        flag[np.unique(plan.dst_idx // nq3)] = True
    return np.flatnonzero(flag), np.flatnonzero(~flag)


class IpcHalo:
    """Peer-memory halo transport for one gs handle (see nk_halo_push /
    nk_halo_combine_wait).  Receive buffer layout (doubles), parity copy c at
    c*buf_len: [own contributions | from neighbour 0 | from neighbour 1 ...]
    exactly as the HaloPlan's buf, so the combine CSR is unchanged."""

    def __init__(self, plan, comm, send_idx, send_slices, device):
        import ctypes
        import struct

        import torch
        from ._lib import check, lib, ptr
        L = lib()
        self.L = L
        nb = plan.neighbors
        if len(nb) > 8:
            raise RuntimeError("IPC halo supports at most 8 neighbours")
        hs = L.nk_ipc_handle_size()
        self.buf_len = max(plan.buf_len, 1)
        self.own_len = len(plan.dst_idx)
        self.buf_ptr = ctypes.c_void_p()
        self.flag_ptr = ctypes.c_void_p()
        hb = (ctypes.c_char * hs)()
        hf = (ctypes.c_char * hs)()
        self.peers = []
        ok = (L.nk_ipc_alloc(2 * self.buf_len * 8, ctypes.byref(self.buf_ptr), hb) == 0 and
              L.nk_ipc_alloc(max(len(nb), 1) * 8, ctypes.byref(self.flag_ptr), hf) == 0)
        if not torch_all_ok(comm, ok):      # every rank leaves together
            self.close()
            raise RuntimeError("IPC allocation failed on some rank")
        # tell each neighbour: my handles, where its contributions go in my buffer,
        # my buffer length and its slot in my flag array
        me = comm.rank
        msgs = {}
        for slot, q in enumerate(nb):
            meta = struct.pack("<qqq", plan.recv_off[q], self.buf_len, slot)
            msgs[q] = bytes(hb) + bytes(hf) + meta
        got = comm.exchange_bytes(msgs)
        n = len(nb)
        self.peer_recv = np.zeros(max(n, 1), dtype=np.uint64)
        self.peer_flag = np.zeros(max(n, 1), dtype=np.uint64)
        self.recv_off = np.zeros(max(n, 1), dtype=np.int64)
        self.recv_len = np.zeros(max(n, 1), dtype=np.int64)
        ok = True
        for i, q in enumerate(nb):
            raw = got[q]
            pb, pf = ctypes.c_void_p(), ctypes.c_void_p()
            if L.nk_ipc_open(raw[:hs], ctypes.byref(pb)) != 0 or \
                    L.nk_ipc_open(raw[hs:2 * hs], ctypes.byref(pf)) != 0:
                ok = False
                break
            off, blen, slot = struct.unpack("<qqq", raw[2 * hs:2 * hs + 24])
            self.peers += [pb, pf]
            self.peer_recv[i] = pb.value
            self.peer_flag[i] = pf.value + 8 * slot
            self.recv_off[i] = off
            self.recv_len[i] = blen
        del me
        if not torch_all_ok(comm, ok):
            self.close()
            raise RuntimeError("IPC peer mapping failed on some rank")
        starts = [0]
        for q in nb:
            a, b = send_slices[q]
            starts.append(b)
        self.send_start = torch.as_tensor(np.asarray(starts, dtype=np.int32), device=device)
        self.send_idx = send_idx
        self.total = int(starts[-1])
        self.nnb = n
        self.epoch = torch.zeros(2, dtype=torch.int64, device=device)

    def own_buffer(self):
        return self.buf_ptr.value

    def push(self, w, st, stream):
        from ._lib import check, ptr
        check(self.L.nk_halo_push(self.nnb, ptr(self.peer_recv), ptr(self.recv_off),
                                  ptr(self.recv_len), ptr(self.peer_flag), ptr(self.send_start),
                                  ptr(self.send_idx), ptr(w), self.total, ptr(self.epoch),
                                  ptr(st), stream), "halo_push")

    def combine(self, h, w, op_code, st, stream):
        from ._lib import check, ptr
        check(self.L.nk_halo_combine_wait(h.nh, ptr(h.src_start), ptr(h.src_idx),
                                          self.buf_ptr.value, self.buf_len, self.own_len,
                                          ptr(h.dst_start), ptr(h.dst_idx), ptr(w), op_code,
                                          self.flag_ptr.value, self.nnb, ptr(self.epoch), ptr(st),
                                          stream), "halo_combine_wait")

    def close(self):
        for p in getattr(self, "peers", []):
            if p.value:
                self.L.nk_ipc_close(p.value)
        self.peers = []
        for p in (self.buf_ptr, self.flag_ptr):
            if p.value:
                self.L.nk_ipc_free(p.value)
                p.value = None


def torch_all_ok(comm, ok):
    """True on every rank iff ok on every rank."""
    import torch
    dev = "cuda" if comm.backend == "nccl" else "cpu"
    t = torch.tensor([1 if ok else 0], dtype=torch.int64, device=dev)
    comm.dist.all_reduce(t, op=comm.dist.ReduceOp.MIN, group=comm.group)
    return bool(int(t.item()))


class IpcBoard:
    """Per-rank scalar board (2 parities x P ranks x 4 doubles) + P flags,
    mapped into every rank (nk_board_allreduce)."""

    def __init__(self, comm, device):
        import ctypes

        import torch
        from ._lib import check, lib
        L = lib()
        self.L, self.comm = L, comm
        P, me = comm.size, comm.rank
        hs = L.nk_ipc_handle_size()
        self.board_ptr, self.flag_ptr = ctypes.c_void_p(), ctypes.c_void_p()
        hb, hf = (ctypes.c_char * hs)(), (ctypes.c_char * hs)()
        self.opened = []
        ok = (L.nk_ipc_alloc(2 * P * 4 * 8, ctypes.byref(self.board_ptr), hb) == 0 and
              L.nk_ipc_alloc(P * 8, ctypes.byref(self.flag_ptr), hf) == 0)
        if not torch_all_ok(comm, ok):
            self.close()
            raise RuntimeError("IPC allocation failed on some rank")
        got = comm.exchange_bytes({q: bytes(hb) + bytes(hf) for q in range(P) if q != me})
        self.boards = np.zeros(P, dtype=np.uint64)
        self.flags_for_me = np.zeros(P, dtype=np.uint64)
        ok = True
        for q in range(P):
            if q == me:
                self.boards[q] = self.board_ptr.value
                self.flags_for_me[q] = self.flag_ptr.value + 8 * me
                continue
            raw = got[q]
            pb, pf = ctypes.c_void_p(), ctypes.c_void_p()
            if L.nk_ipc_open(raw[:hs], ctypes.byref(pb)) != 0 or \
                    L.nk_ipc_open(raw[hs:2 * hs], ctypes.byref(pf)) != 0:
                ok = False
                break
            self.opened += [pb, pf]
            self.boards[q] = pb.value
            self.flags_for_me[q] = pf.value + 8 * me
        if not torch_all_ok(comm, ok):
            self.close()
            raise RuntimeError("IPC peer mapping failed on some rank")
        self.epoch = torch.zeros(2, dtype=torch.int64, device=device)

    def allreduce_(self, t):
        from ._lib import check, ptr, stream_ptr
        check(self.L.nk_board_allreduce(self.comm.size, self.comm.rank, ptr(t), t.numel(),
                                        ptr(self.boards), ptr(self.flags_for_me),
                                        self.board_ptr.value, self.flag_ptr.value,
                                        ptr(self.epoch), stream_ptr()), "board_allreduce")

    def close(self):
        for p in getattr(self, "opened", []):
            if p.value:
                self.L.nk_ipc_close(p.value)
        self.opened = []
        for p in (self.board_ptr, self.flag_ptr):
            if p.value:
                self.L.nk_ipc_free(p.value)
                p.value = None
