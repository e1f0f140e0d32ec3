"""Oracle: gather-scatter QQ^T in canonical order.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates SPEC.md:192-210 (gs_setup / gs_op) and SPEC.md:205, 250 (canonical
accumulation order: ascending rank, then ascending local index), with
SPEC.md:195 (ids held once are singletons) and SPEC.md:198 (all-zero ids ->
identity).  The reduction is an explicit sequential left fold per id, so the
floating-point association is exactly the canonical order.
"""

import numpy as np

OPS = ("+", "*", "min", "max")


def _fold(op, acc, v):
    if op == "+":
        return acc + v
    if op == "*":
        return acc * v
    if op == "min":
        return np.minimum(acc, v)
    if op == "max":
        return np.maximum(acc, v)
    raise ValueError(f"unknown op {op!r}")


def local_plan(ids):
    """(perm, seg_start) for one rank: ids with multiplicity >= 2, segments in
    ascending id order, members in ascending local index."""
    ids = np.asarray(ids, dtype=np.int64).ravel()
    order = np.argsort(ids, kind="stable")
    s = ids[order]
    nz = s != 0
    order, s = order[nz], s[nz]
    if len(s) == 0:
        return np.zeros(0, np.int64), np.zeros(1, np.int64)
    start = np.flatnonzero(np.r_[True, s[1:] != s[:-1]])
    cnt = np.diff(np.r_[start, len(s)])
    keep = cnt >= 2
    segs_start, segs_cnt = start[keep], cnt[keep]
    perm = np.concatenate([order[a:a + c] for a, c in zip(segs_start, segs_cnt)]) \
        if len(segs_start) else np.zeros(0, np.int64)
    seg_start = np.r_[0, np.cumsum(segs_cnt)].astype(np.int64)
    return perm.astype(np.int64), seg_start


def gs_op_plan(perm, seg_start, w, op="+", precision=64):
    """Apply a local plan: sequential fold in plan order; writes back.
    precision 32 folds in float32 (SPEC.md:202's 32-bit gs)."""
    w = np.array(w, dtype=np.float32 if precision == 32 else np.float64, copy=True)
    flat = w.reshape(-1)
    if len(seg_start) <= 1:
        return w
    cnt = np.diff(seg_start)
    acc = flat[perm[seg_start[:-1]]].copy()
    for p in range(1, int(cnt.max())):
        act = cnt > p
        acc[act] = _fold(op, acc[act], flat[perm[seg_start[:-1][act] + p]])
    seg_of = np.repeat(np.arange(len(cnt)), cnt)
    flat[perm] = acc[seg_of]
    return w


def gs_op(ids, w, op="+", precision=64):
    """Single-rank QQ^T."""
    ids = np.asarray(ids).ravel()
    if np.asarray(w).size != ids.size:
        raise ValueError("contract error: field length mismatch")
    perm, seg = local_plan(ids)
    return gs_op_plan(perm, seg, w, op, precision)


def gs_op_multi(ids_per_rank, w_per_rank, op="+"):
    """Simulated P-rank QQ^T: every id reduced over ALL holders in ascending
    (rank, local index) order."""
    P = len(ids_per_rank)
    rk = np.concatenate([np.full(len(np.ravel(i)), r) for r, i in enumerate(ids_per_rank)])
    li = np.concatenate([np.arange(len(np.ravel(i))) for i in ids_per_rank])
    gid = np.concatenate([np.ravel(i) for i in ids_per_rank]).astype(np.int64)
    val = np.concatenate([np.ravel(np.asarray(v, dtype=np.float64)) for v in w_per_rank])
    # canonical order: (gid, rank, local index); ranks are concatenated in order
    out = gs_op(gid, val, op)
    offs = np.r_[0, np.cumsum([len(np.ravel(i)) for i in ids_per_rank])]
    del rk, li
    return [out[offs[r]:offs[r + 1]].reshape(np.shape(w_per_rank[r])) for r in range(P)]


def dense_Q(ids):
    """Explicit 0/1 Q (n_local x n_unique) for the dense oracle.
    Singleton/zero ids get their own column."""
    ids = np.asarray(ids).ravel()
    n = len(ids)
    key = ids.copy().astype(np.int64)
    zero = key == 0
    key[zero] = -(np.arange(n)[zero] + 1)
    u, inv = np.unique(key, return_inverse=True)
    Q = np.zeros((n, len(u)))
    Q[np.arange(n), inv] = 1.0
    return Q


def multiplicity(ids):
    ids = np.asarray(ids).ravel()
    u, inv, cnt = np.unique(ids, return_inverse=True, return_counts=True)
    m = cnt[inv].astype(np.float64)
    m[ids == 0] = 1.0
    return m
