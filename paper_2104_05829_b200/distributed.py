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
The exchanged values are the per-rank partial sums of the local gs; the
receiver folds the holders' partials in ascending rank order (own partial at
its rank position), so every rank computes bit-identical totals.
"""

import numpy as np


class RankComm:
    """Collective context for one rank.

    group: a torch.distributed ProcessGroup (None = default group).
    staging: 'device' exchanges device buffers directly (NCCL); 'host' stages
    them through host memory (the paper's host-staged variant; used with gloo
    when several ranks share one GPU in tests)."""

    def __init__(self, group=None, staging=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.backend = backend
        self.staging = staging or ("device" if backend == "nccl" else "host")

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

    def allreduce_sum_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def barrier(self):
        self.dist.barrier(group=self.group)

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
    holders     list of holder-rank arrays per halo id (ascending)
    neighbors   sorted neighbour ranks; ngh = len(neighbors)
    rep         local index of the first local copy of each halo id
    dst_start/dst_idx   CSR: all local copies of each halo id (ascending)
    send[q]     positions (into hids) sent to / received from neighbour q
    src_start/src_idx   CSR into buf = [own partials (nh) | recv_q0 | recv_q1 ...]
                        listing the holders' partials in ascending rank order
    """


def _face_point_mask(nq):
    r = np.arange(nq)
    on = (r == 0) | (r == nq - 1)
    return (on[:, None, None] | on[None, :, None] | on[None, None, :]).ravel()


def build_halo_plan(ids, comm, nq=None):
    """Collective discovery of rank-shared ids (see module doc)."""
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
    parts = [cand[owner == q] for q in range(P)]
    got = comm.alltoallv_int64(parts)
    # owner side: (id, holder-rank) pairs -> bitmask per id held by >= 2 ranks
    gid = np.concatenate(got) if got else np.zeros(0, np.int64)
    src = np.concatenate([np.full(len(g), q, dtype=np.int64) for q, g in enumerate(got)])
    replies = [np.zeros(0, np.int64)] * P
    if len(gid):
        o = np.lexsort((src, gid))
        gid, src = gid[o], src[o]
        u, start, cnt = np.unique(gid, return_index=True, return_counts=True)
        bits = np.zeros(len(u), dtype=np.int64)
        np.bitwise_or.at(bits, np.repeat(np.arange(len(u)), cnt), np.left_shift(1, src))
        shared = cnt >= 2
        us, bs = u[shared], bits[shared]
        rep_parts = [[] for _ in range(P)]
        for q in range(P):
            sel = (bs >> q) & 1 == 1
            rep_parts[q] = np.stack([us[sel], bs[sel]], axis=1).ravel()
        replies = rep_parts
    back = comm.alltoallv_int64(replies)
    rec = np.concatenate([b.reshape(-1, 2) for b in back]) if back else np.zeros((0, 2), np.int64)
    o = np.argsort(rec[:, 0], kind="stable") if len(rec) else np.zeros(0, np.int64)
    rec = rec[o]
    plan = HaloPlan()
    plan.rank, plan.size = me, P
    plan.hids = rec[:, 0].copy()
    masks = rec[:, 1].copy()
    nh = len(plan.hids)
    plan.holders = [np.flatnonzero((int(m) >> np.arange(P)) & 1) for m in masks]
    nb = sorted({int(q) for h in plan.holders for q in h if q != me})
    plan.neighbors = nb
    plan.ngh = len(nb)
    # local copies of every halo id (ascending local index)
    order = np.argsort(ids, kind="stable")
    sids = ids[order]
    lo = np.searchsorted(sids, plan.hids, side="left")
    hi = np.searchsorted(sids, plan.hids, side="right")
    if np.any(hi <= lo):
        raise RuntimeError("halo id without a local copy (inconsistent discovery)")
    plan.dst_start = np.r_[0, np.cumsum(hi - lo)].astype(np.int64)
    plan.dst_idx = np.concatenate([order[a:b] for a, b in zip(lo, hi)]) if nh else \
        np.zeros(0, np.int64)
    plan.rep = order[lo] if nh else np.zeros(0, np.int64)
    # per-neighbour positions in hids, ascending id order on both sides
    plan.send = {}
    for q in nb:
        plan.send[q] = np.array([t for t in range(nh) if q in set(plan.holders[t])],
                                dtype=np.int64)
    # combine CSR into buf = [own | recv_q (for q in neighbors)]
    recv_off, off = {}, nh
    for q in nb:
        recv_off[q] = off
        off += len(plan.send[q])
    plan.buf_len = off
    plan.recv_off = recv_off
    pos_in_q = {q: {int(t): i for i, t in enumerate(plan.send[q])} for q in nb}
    src_start, src_idx = [0], []
    for t in range(nh):
        for q in plan.holders[t]:
            q = int(q)
            src_idx.append(t if q == me else recv_off[q] + pos_in_q[q][t])
        src_start.append(len(src_idx))
    plan.src_start = np.asarray(src_start, dtype=np.int64)
    plan.src_idx = np.asarray(src_idx, dtype=np.int64)
    return plan


def boundary_elements(plan, n_elem, nq3):
    """Elements holding at least one halo id (evaluated first)."""
    flag = np.zeros(n_elem, dtype=bool)
    if len(plan.dst_idx):
        flag[np.unique(plan.dst_idx // nq3)] = True
    return np.flatnonzero(flag), np.flatnonzero(~flag)
