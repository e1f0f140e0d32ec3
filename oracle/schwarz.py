"""Oracle: FDM local solves and overlapping Schwarz (ASM / RAS) smoothing.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates SPEC.md:410-418 (fdm_local_solve), 499-507 (schwarz_smooth),
462-464 (SmootherConfig kinds asm, ras, cheby_asm, cheby_ras) and PAPER.md:
298-313 (one-element overlap, (N+3)^3 extended subdomains, FDM cost
12E(N+3)^4, ASM weighted by the counting function, RAS keeps its own data).
No reference code exists; the SPEC leaves these choices open, frozen here
(DESIGN.md "Schwarz smoother"):

Extended subdomain.  Element e's box has (N+3)^3 points (i', j', k'), i' = i+1.
  * interior (i', j', k') in [1, N+1]^3: e's own point (i, j, k);
  * face extension (exactly one coordinate 0 or N+2): the point ONE LAYER
    INSIDE the face neighbour -- the neighbour's point adjacent (along the
    neighbour's face normal) to the face point e shares with it.  Face
    neighbours are found from the global ids (two faces are neighbours when
    their (N+1)^2 id sets coincide), so HEXMESH meshes and periodic boxes work
    unchanged.  No neighbour -> no extension point;
  * edges / corners of the extended box: never sampled (zero input, output
    discarded).
  The extended input of a continuous L-vector r is r sampled at those points;
  the "dedicated gs handle" of SPEC.md:504 is gs over extended ids (the global
  id of each sampled point, 0 where nothing is sampled).

FDM surrogate (per element, per reference direction d).  h_d = mean distance
between the element's two opposite d-faces (over the (N+1)^2 face point
pairs).  The 1-D problem lives on three equal elements of length h_d
(left neighbour, own, right neighbour; K_el = (2/h) D^T W D, M_el = (h/2) W,
W = GLL weights) assembled on 3N+1 points and restricted to the N+3 points
{left N-1, own 0..N, right 1}.  Side kinds: 'nbr' (neighbour exists: left /
right element assembled in), 'neu' (no neighbour, face not masked: that
element left out, extension point dropped), 'dir' (no neighbour, face masked:
extension and face point dropped).  Dropped points are removed from the
generalised eigenproblem K S = M S Lambda (S^T M S = I) and carry
lambda = +inf (their output is exactly 0).  3-D:
    u = (Sz x Sy x Sx) diag(1 / (lam0 (Lx + Ly + Lz) + lam1)) (Sz x Sy x Sx)^T r
Pure Neumann surrogate (no dropped point on any side, lam1 = 0): each 1-D
spectrum is shifted by eps/3 with eps = 1e-8 max(Lambda).

Smoothers (z = S r, r assembled and masked):
  * asm: z = mask * W_ext * QQ^T_ext(u_ext) restricted to own points, with
    W_ext = 1 / (number of extended boxes holding the point) -- exchange and
    add with the counting weight;
  * ras: z = mask * (1/mult) * QQ^T(u_ext restricted to own points) -- each
    element keeps its own (interior) data, no overlap sum; the
    1/mult average keeps z continuous on shared interfaces.
"""

import numpy as np

from . import gs as ogs

FACE_AXES = ((0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1))   # (axis, side) in x-,x+,y-,...


def _face_slice(nq, axis, side):
    """Index tuple selecting a face of an (E, nq, nq, nq) [e][k][j][i] array
    and the one-layer-inward slice; both (E, nq, nq) over the two tangential
    indices in (slow, fast) order."""
    pos = 0 if side == 0 else nq - 1
    inw = 1 if side == 0 else nq - 2
    def sl(p):
        s = [slice(None)] * 4
        s[3 - axis] = p        # axis 0 = i (last index), 1 = j, 2 = k
        return tuple(s)
    return sl(pos), sl(inw)


def face_source_map(ids, E, N):
    """fmap[e, f, a, b] = local index (into the flat L-vector) of the point
    one layer inside the face neighbour across face f of element e, at the
    position matching e's face point (a, b); -1 without a neighbour.
    f in x-, x+, y-, y+, z-, z+; (a, b) the tangential indices (slow, fast)."""
    nq = N + 1
    ids = np.asarray(ids, dtype=np.int64).reshape(E, nq, nq, nq)
    loc = np.arange(E * nq ** 3, dtype=np.int64).reshape(E, nq, nq, nq)
    fid, finw = [], []
    for axis, side in FACE_AXES:
        fs, ins = _face_slice(nq, axis, side)
        fid.append(ids[fs].reshape(E, nq * nq))
        finw.append(loc[ins].reshape(E, nq * nq))
    fid = np.stack(fid, 1).reshape(E * 6, nq * nq)            # rows: (e, f)
    finw = np.stack(finw, 1).reshape(E * 6, nq * nq)
    srt = np.sort(fid, axis=1)
    _, grp, cnt = np.unique(srt, axis=0, return_inverse=True, return_counts=True)
    grp = grp.ravel()
    fmap = np.full((E * 6, nq * nq), -1, dtype=np.int64)
    if np.any(cnt > 2):
        raise ValueError("a face id set is held by more than two element faces")
    order = np.argsort(grp, kind="stable")
    g = grp[order]
    starts = np.flatnonzero(np.r_[True, g[1:] != g[:-1]])
    pairs = [(order[s], order[s + 1]) for s in starts if s + 1 < len(g) and g[s + 1] == g[s]]
    for r0, r1 in pairs:
        for a, b in ((r0, r1), (r1, r0)):
            # position in b's face of each of a's face ids: the q-th smallest
            # id of a's face (stable order for repeated ids on periodic
            # single-element axes) sits at b's q-th smallest
            ob = np.argsort(fid[b], kind="stable")
            rank = np.empty(nq * nq, dtype=np.int64)
            rank[np.argsort(fid[a], kind="stable")] = np.arange(nq * nq)
            fmap[a] = finw[b][ob[rank]]
    return fmap.reshape(E, 6, nq, nq)


def side_kinds(fmap, mask, E, N):
    """kinds[e, f] in {'nbr', 'neu', 'dir'}."""
    nq = N + 1
    mask = np.asarray(mask).reshape(E, nq, nq, nq)
    kinds = np.empty((E, 6), dtype=object)
    for f, (axis, side) in enumerate(FACE_AXES):
        fs, _ = _face_slice(nq, axis, side)
        masked = np.all(mask[fs].reshape(E, -1) == 0, axis=1)
        has = fmap[:, f, 0, 0] >= 0
        kinds[:, f] = np.where(has, "nbr", np.where(masked, "dir", "neu"))
    return kinds


def element_lengths(xyz, E, N):
    """h[e, d]: mean distance between the element's two opposite d-faces."""
    nq = N + 1
    X = np.asarray(xyz).reshape(3, E, nq, nq, nq)
    h = np.zeros((E, 3))
    for d in range(3):
        lo, _ = _face_slice(nq, d, 0)
        hi, _ = _face_slice(nq, d, 1)
        diff = np.stack([X[c][hi] - X[c][lo] for c in range(3)])
        h[:, d] = np.mean(np.sqrt(np.sum(diff ** 2, axis=0)).reshape(E, -1), axis=1)
    return h


def fdm_1d(D, w, h, left, right):
    """(S, lam) of the extended 1-D problem: S (N+3, N+3) with S^T M S = I on
    kept points, lam (N+3,) with +inf for dropped points."""
    N = len(w) - 1
    K1 = (2.0 / h) * D.T @ (w[:, None] * D)
    M1 = (h / 2.0) * w
    n3 = 3 * N + 1
    K = np.zeros((n3, n3))
    M = np.zeros(n3)
    use = [left == "nbr", True, right == "nbr"]
    for el in range(3):
        if use[el]:
            s = el * N
            K[s:s + N + 1, s:s + N + 1] += K1
            M[s:s + N + 1] += M1
    sel = np.arange(N - 1, 2 * N + 2)                    # N+3 points
    K = K[np.ix_(sel, sel)]
    M = M[sel]
    keep = np.ones(N + 3, dtype=bool)
    if left != "nbr":
        keep[0] = False
        if left == "dir":
            keep[1] = False
    if right != "nbr":
        keep[N + 2] = False
        if right == "dir":
            keep[N + 1] = False
    kk = np.flatnonzero(keep)
    Mh = 1.0 / np.sqrt(M[kk])
    lam_k, V = np.linalg.eigh(Mh[:, None] * K[np.ix_(kk, kk)] * Mh[None, :])
    S = np.zeros((N + 3, N + 3))
    lam = np.full(N + 3, np.inf)
    S[kk, :len(kk)] = Mh[:, None] * V
    lam[:len(kk)] = lam_k
    drop = np.flatnonzero(~keep)
    for c, p in enumerate(drop):
        S[p, len(kk) + c] = 1.0
    return S, lam, keep


class FDM:
    pass


def fdm_setup(mesh_xyz, ids, mask, E, N, D, w, lam0=1.0, lam1=0.0):
    f = FDM()
    f.E, f.N, f.nqe = E, N, N + 3
    f.fmap = face_source_map(ids, E, N)
    f.kinds = side_kinds(f.fmap, mask, E, N)
    f.h = element_lengths(mesh_xyz, E, N)
    f.lam0, f.lam1 = lam0, lam1
    f.S = np.zeros((E, 3, N + 3, N + 3))
    f.lam = np.zeros((E, 3, N + 3))
    f.keep = np.zeros((E, 3, N + 3), dtype=bool)
    for e in range(E):
        for d in range(3):
            S, lam, keep = fdm_1d(D, w, f.h[e, d], f.kinds[e, 2 * d], f.kinds[e, 2 * d + 1])
            f.S[e, d], f.lam[e, d], f.keep[e, d] = S, lam, keep
        if lam1 == 0.0 and all(f.kinds[e, 2 * d] == "neu" and f.kinds[e, 2 * d + 1] == "neu"
                               for d in range(3)):
            # pure-Neumann surrogate: shift by eps = 1e-8 max(Lambda)
            fin = np.isfinite(f.lam[e])
            eps = 1e-8 * float(np.sum(np.max(np.where(fin, f.lam[e], 0.0), axis=1)))
            f.lam[e] = np.where(fin, f.lam[e] + eps / 3.0, np.inf)
    # extended ids and source indices
    nq, nqe = N + 1, N + 3
    ids = np.asarray(ids, dtype=np.int64).ravel()
    src = np.full((E, nqe, nqe, nqe), -1, dtype=np.int64)
    loc = np.arange(E * nq ** 3).reshape(E, nq, nq, nq)
    src[:, 1:nq + 1, 1:nq + 1, 1:nq + 1] = loc
    for fi, (axis, side) in enumerate(FACE_AXES):
        p = 0 if side == 0 else nqe - 1
        s = [slice(None), slice(1, nq + 1), slice(1, nq + 1), slice(1, nq + 1)]
        s[3 - axis] = p
        src[tuple(s)] = f.fmap[:, fi]
    f.src = src.reshape(-1)
    f.ext_ids = np.where(f.src >= 0, ids[np.maximum(f.src, 0)], 0)
    cnt = ogs.gs_op(f.ext_ids, (f.src >= 0).astype(np.float64))
    own = src[:, 1:nq + 1, 1:nq + 1, 1:nq + 1].reshape(-1)
    order = np.argsort(own)
    Wext = np.zeros(E * nq ** 3)
    Wext[own[order]] = 1.0 / cnt.reshape(E, nqe, nqe, nqe)[:, 1:nq + 1, 1:nq + 1, 1:nq + 1] \
        .reshape(-1)[order]
    f.Wext = Wext
    return f


def extend(f, r):
    """r_ext[e] (E, nqe, nqe, nqe) sampled from the L-vector r."""
    r = np.asarray(r).ravel()
    out = np.where(f.src >= 0, r[np.maximum(f.src, 0)], 0.0)
    return out.reshape(f.E, f.nqe, f.nqe, f.nqe)


def fdm_solve(f, r_ext):
    """u_ext = S inv S^T r_ext per element."""
    Sx, Sy, Sz = f.S[:, 0], f.S[:, 1], f.S[:, 2]
    t = np.einsum("eia,ekji->ekja", Sx, r_ext)          # S_x^T along i
    t = np.einsum("ejb,ekja->ekba", Sy, t)
    t = np.einsum("ekc,ekba->ecba", Sz, t)
    t = t * np.stack([inverse_spectrum(f, e) for e in range(f.E)])
    t = np.einsum("ekc,ecba->ekba", Sz, t)
    t = np.einsum("ejb,ekba->ekja", Sy, t)
    return np.einsum("eia,ekja->ekji", Sx, t)


def inverse_spectrum(f, e):
    """1 / (lam0 (Lz + Ly + Lx) + lam1) on the (N+3)^3 modes [c][b][a];
    0 on modes involving a dropped point (lambda = inf)."""
    lx, ly, lz = f.lam[e]
    fin = np.isfinite(lz)[:, None, None] & np.isfinite(ly)[None, :, None] & \
        np.isfinite(lx)[None, None, :]
    sx, sy, sz = (np.where(np.isfinite(v), v, 0.0) for v in (lx, ly, lz))
    den = f.lam0 * (sz[:, None, None] + sy[None, :, None] + sx[None, None, :]) + f.lam1
    return np.where(fin, 1.0 / np.where(fin, den, 1.0), 0.0)


def surrogate_dense(f, e):
    """Dense surrogate operator of element e on its kept extended points
    (for the dense-inverse oracle of SPEC.md:415): K3 and M3 from the 1-D
    pieces, restricted to kept points."""
    mats = []
    for d in range(3):
        S, lam, keep = f.S[e, d], f.lam[e, d], f.keep[e, d]
        kk = np.flatnonzero(keep)
        nk = len(kk)
        Sk = S[np.ix_(kk, np.arange(nk))]
        Minv = Sk @ Sk.T                         # M^-1 on kept points
        M = np.linalg.inv(Minv)
        K = M @ Sk @ np.diag(lam[:nk]) @ Sk.T @ M
        mats.append((kk, K, M))
    (kx, Kx, Mx), (ky, Ky, My), (kz, Kz, Mz) = mats
    A = f.lam0 * (np.kron(Kz, np.kron(My, Mx)) + np.kron(Mz, np.kron(Ky, Mx)) +
                  np.kron(Mz, np.kron(My, Kx))) + f.lam1 * np.kron(Mz, np.kron(My, Mx))
    nqe = f.nqe
    flat = (kz[:, None, None] * nqe * nqe + ky[None, :, None] * nqe + kx[None, None, :]).ravel()
    return flat, A


def schwarz_smooth(f, kind, r, ids, mask):
    """z = S r for kind in {'asm', 'ras'}."""
    nq, nqe, E = f.N + 1, f.nqe, f.E
    u = fdm_solve(f, extend(f, r))
    mask = np.asarray(mask).ravel()
    if kind == "asm":
        s = ogs.gs_op(f.ext_ids, u.reshape(-1)).reshape(E, nqe, nqe, nqe)
        z = s[:, 1:nq + 1, 1:nq + 1, 1:nq + 1].reshape(-1)
        return mask * f.Wext * z
    if kind == "ras":
        z = u[:, 1:nq + 1, 1:nq + 1, 1:nq + 1].reshape(-1)
        return mask * ogs.gs_op(ids, z) / ogs.multiplicity(ids)
    raise ValueError(f"unknown Schwarz kind {kind!r}")


def fdm_flops(N, E):
    """12 E (N+3)^4 (FDM cost ~ 12E(N+3)^4)."""
    return 12 * E * (N + 3) ** 4
