"""Oracle: box meshes, geometric factors, global ids, Dirichlet masks, HEXMESH.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates SPEC.md:96-170 (no reference code exists for the mesh module):
  * build_box_mesh        SPEC.md:118-126  (trilinear-then-deformed GLL points)
  * geometric_factors     SPEC.md:128-136, PAPER.md:1177-1180 (dx/dr = D_q x),
                          PAPER.md:1256-1263 (G), PAPER.md:1213-1218 (B = rho J)
  * assign_global_ids     SPEC.md:138-146  (ids by sorted coordinate order)
  * Dirichlet mask
  * HEXMESH v1

Frozen decisions:
  * Element order e = ex + nx*(ey + ny*ez); point order i fastest, then j, k.
  * Global ids of a generated box are assigned by sorting the points'
    UNDEFORMED lattice coordinates (gx, gy, gz) = (ex*N+i, ey*N+j, ez*N+k)
    (wrapped modulo nx*N on periodic axes) lexicographically by (z, y, x) and
    numbering unique points 1, 2, ... in that order.  The deformation is a
    bijection, so coincidence classes are unchanged, and the integer lattice
    makes the numbering free of floating-point ties.  Meshes read from files
    use assign_global_ids() on physical coordinates (tolerance snapping).
  * The mesh keeps the FULL numbering (every id nonzero; SPEC.md:126 counts
    interior points).  singleton_ids() zeroes ids held once;
    gs_setup treats ids held once as singletons either way.
  * Deformation 'sine' (amplitude a, default 0.05), boundary-preserving:
        x' = x + a Lx sin(2 pi X) sin(pi Y) sin(pi Z)
        y' = y + a Ly sin(pi X) sin(2 pi Y) sin(pi Z)
        z' = z + a Lz sin(pi X) sin(pi Y) sin(2 pi Z)
    with X, Y, Z the coordinates normalised to [0, 1] over the box.
  * G is stored element-blocked [E][6][(N+1)^3] in the order
    G11, G12, G13, G22, G23, G33.
"""

import numpy as np

from .basis import Basis

FACES = ("x-", "x+", "y-", "y+", "z-", "z+")


class InvertedElementError(ValueError):
    pass


class DegenerateElementError(ValueError):
    pass


def normalize_bc(bc):
    """bc: str for all faces, or dict face->kind, or 6-sequence in FACES order.
    kinds: 'dirichlet' | 'neumann' | 'periodic'."""
    if isinstance(bc, str):
        out = {f: bc for f in FACES}
    elif isinstance(bc, dict):
        out = {f: bc.get(f, "neumann") for f in FACES}
    else:
        bc = list(bc)
        out = dict(zip(FACES, bc))
    for a in range(3):
        lo, hi = out[FACES[2 * a]], out[FACES[2 * a + 1]]
        if (lo == "periodic") != (hi == "periodic"):
            raise ValueError(f"periodic bc must pair both faces of axis {a}")
    return out


def deform_sine(X, Y, Z, amp, L):
    s = np.sin
    p = np.pi
    dx = amp * L[0] * s(2 * p * X) * s(p * Y) * s(p * Z)
    dy = amp * L[1] * s(p * X) * s(2 * p * Y) * s(p * Z)
    dz = amp * L[2] * s(p * X) * s(p * Y) * s(2 * p * Z)
    return dx, dy, dz


class BoxMesh:
    pass


def box_coordinates(extent, counts, N, origin=(0.0, 0.0, 0.0), deformation=None,
                    elements=None):
    """GLL point coordinates, shape (3, E, nq, nq, nq) [c][e][k][j][i]."""
    nx, ny, nz = counts
    nq = N + 1
    r = Basis.get(N).nodes
    E = nx * ny * nz
    el = np.arange(E) if elements is None else np.asarray(elements)
    ex, ey, ez = el % nx, (el // nx) % ny, el // (nx * ny)
    h = [extent[0] / nx, extent[1] / ny, extent[2] / nz]
    t = 0.5 * (r + 1.0)
    X = origin[0] + (ex[:, None] + t[None, :]) * h[0]      # (E, nq) along i
    Y = origin[1] + (ey[:, None] + t[None, :]) * h[1]
    Z = origin[2] + (ez[:, None] + t[None, :]) * h[2]
    shape = (len(el), nq, nq, nq)
    x = np.broadcast_to(X[:, None, None, :], shape).copy()
    y = np.broadcast_to(Y[:, None, :, None], shape).copy()
    z = np.broadcast_to(Z[:, :, None, None], shape).copy()
    if deformation is not None:
        if callable(deformation):
            x, y, z = deformation(x, y, z)
        else:
            kind, amp = deformation
            if kind != "sine":
                raise ValueError(f"unknown deformation {kind!r}")
            Xn = (x - origin[0]) / extent[0]
            Yn = (y - origin[1]) / extent[1]
            Zn = (z - origin[2]) / extent[2]
            dx, dy, dz = deform_sine(Xn, Yn, Zn, amp, extent)
            x, y, z = x + dx, y + dy, z + dz
    return np.stack([x, y, z])


def lattice_ids(counts, N, periodic=(False, False, False)):
    """Global ids by lexicographic (z, y, x) sort of the integer lattice
    coordinates of every local point (frozen decision, see module doc)."""
    nx, ny, nz = counts
    nq = N + 1
    E = nx * ny * nz
    el = np.arange(E)
    ex, ey, ez = el % nx, (el // nx) % ny, el // (nx * ny)
    ii = np.arange(nq)
    gx = (ex[:, None] * N + ii[None, :])
    gy = (ey[:, None] * N + ii[None, :])
    gz = (ez[:, None] * N + ii[None, :])
    Lx, Ly, Lz = nx * N, ny * N, nz * N
    if periodic[0]:
        gx = gx % Lx
    if periodic[1]:
        gy = gy % Ly
    if periodic[2]:
        gz = gz % Lz
    shape = (E, nq, nq, nq)
    GX = np.broadcast_to(gx[:, None, None, :], shape).ravel()
    GY = np.broadcast_to(gy[:, None, :, None], shape).ravel()
    GZ = np.broadcast_to(gz[:, :, None, None], shape).ravel()
    return ids_from_keys(GX, GY, GZ)


def ids_from_keys(kx, ky, kz):
    """1-based rank of each (kz, ky, kx) triple among the unique triples."""
    order = np.lexsort((kx, ky, kz))
    sx, sy, sz = kx[order], ky[order], kz[order]
    new = np.ones(len(order), dtype=bool)
    new[1:] = (sx[1:] != sx[:-1]) | (sy[1:] != sy[:-1]) | (sz[1:] != sz[:-1])
    rank = np.cumsum(new)
    ids = np.empty(len(order), dtype=np.int64)
    ids[order] = rank
    return ids


def assign_global_ids(coords, tol_rel=1e-10):
    """Generic id discovery from physical coordinates:
    snap to a grid of spacing tol_rel * (domain diameter), sort (z, y, x),
    number unique points from 1.  coords: (3, n)."""
    c = np.asarray(coords, dtype=np.float64).reshape(3, -1)
    lo = c.min(axis=1)
    diam = float(np.linalg.norm(c.max(axis=1) - lo))
    tol = tol_rel * max(diam, 1e-300)
    k = np.rint((c - lo[:, None]) / tol).astype(np.int64)
    return ids_from_keys(k[0], k[1], k[2])


def singleton_ids(ids):
    """Zero the ids that occur exactly once."""
    ids = np.asarray(ids)
    u, inv, cnt = np.unique(ids, return_inverse=True, return_counts=True)
    out = ids.copy()
    out[cnt[inv] == 1] = 0
    out[ids == 0] = 0
    return out


def geometric_factors(xyz, D, w):
    """Per element factors from coordinates.

    xyz: (3, E, nq, nq, nq); D: (nq, nq) D-hat; w: (nq,) GLL weights.
    Returns J (E,nq,nq,nq), metrics rx[q][p] = dr_q/dx_p (3,3,E,nq,nq,nq),
    G (E, 6, nq, nq, nq), B (E, nq, nq, nq).
    """
    xyz = np.asarray(xyz, dtype=np.float64)
    # dx_p/dr_q via D_q x_p: r along i, s along j, t along k
    dr = np.einsum("im,cekjm->cekji", D, xyz)
    ds = np.einsum("jm,cekmi->cekji", D, xyz)
    dt = np.einsum("km,cemji->cekji", D, xyz)
    Jm = np.stack([dr, ds, dt], axis=1)                # Jm[p][q] = dx_p/dr_q
    a = Jm
    J = (a[0, 0] * (a[1, 1] * a[2, 2] - a[1, 2] * a[2, 1])
         - a[0, 1] * (a[1, 0] * a[2, 2] - a[1, 2] * a[2, 0])
         + a[0, 2] * (a[1, 0] * a[2, 1] - a[1, 1] * a[2, 0]))
    if np.any(np.abs(J) < 1e-14):
        e = int(np.argwhere(np.abs(J) < 1e-14)[0][0])
        raise DegenerateElementError(f"degenerate element {e}: |J| < 1e-14")
    # inverse: rx[q][p] = cofactor(p,q)/J
    cof = np.empty_like(a)
    for p in range(3):
        for q in range(3):
            p1, p2 = [t for t in range(3) if t != p]
            q1, q2 = [t for t in range(3) if t != q]
            minor = a[p1, q1] * a[p2, q2] - a[p1, q2] * a[p2, q1]
            cof[p, q] = ((-1) ** (p + q)) * minor
    rx = np.empty_like(a)
    for q in range(3):
        for p in range(3):
            rx[q, p] = cof[p, q] / J
    rho = w[:, None, None] * w[None, :, None] * w[None, None, :]   # [k][j][i]
    wJ = rho[None] * J
    pairs = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
    G = np.stack([(rx[m, 0] * rx[n, 0] + rx[m, 1] * rx[n, 1] + rx[m, 2] * rx[n, 2]) * wJ
                  for m, n in pairs], axis=1)
    B = wJ
    return J, rx, G, B


def dirichlet_mask(counts, N, bc):
    """0 on gridpoints of Dirichlet faces, else 1; shape (E, nq, nq, nq)."""
    bc = normalize_bc(bc)
    nx, ny, nz = counts
    nq = N + 1
    E = nx * ny * nz
    el = np.arange(E)
    ex, ey, ez = el % nx, (el // nx) % ny, el // (nx * ny)
    m = np.ones((E, nq, nq, nq))
    if bc["x-"] == "dirichlet":
        m[ex == 0, :, :, 0] = 0
    if bc["x+"] == "dirichlet":
        m[ex == nx - 1, :, :, N] = 0
    if bc["y-"] == "dirichlet":
        m[ey == 0, :, 0, :] = 0
    if bc["y+"] == "dirichlet":
        m[ey == ny - 1, :, N, :] = 0
    if bc["z-"] == "dirichlet":
        m[ez == 0, 0, :, :] = 0
    if bc["z+"] == "dirichlet":
        m[ez == nz - 1, N, :, :] = 0
    return m


def build_box_mesh(extent, counts, N, bc="dirichlet", deformation=None,
                   origin=(0.0, 0.0, 0.0)):
    """Oracle box mesh. Returns a BoxMesh with numpy fields:
    xyz (3,E,nq,nq,nq), G (E,6,nq,nq,nq), B, J, ids (E*nq^3,), mask."""
    counts = tuple(int(c) for c in counts)
    if min(counts) < 1:
        raise ValueError("counts must be >= 1")
    bcn = normalize_bc(bc)
    basis = Basis.get(N)
    xyz = box_coordinates(extent, counts, N, origin, deformation)
    J, rx, G, B = geometric_factors(xyz, basis.diff, basis.weights)
    if np.any(J <= 0):
        e = int(np.argwhere(J <= 0)[0][0])
        raise InvertedElementError(f"inverted element {e}")
    periodic = tuple(bcn[FACES[2 * a]] == "periodic" for a in range(3))
    m = BoxMesh()
    m.N, m.nq, m.counts, m.extent, m.origin = N, N + 1, counts, tuple(extent), tuple(origin)
    m.E = counts[0] * counts[1] * counts[2]
    m.bc, m.deformation = bcn, deformation
    m.xyz, m.J, m.G, m.B = xyz, J, G, B
    m.ids = lattice_ids(counts, N, periodic)
    m.mask = dirichlet_mask(counts, N, bcn)
    m.basis = basis
    return m


# ---------------------------------------------------------------- HEXMESH v1

def write_hexmesh(path, xyz, ids, masks=None):
    """header, (N+1)^3 'x y z' lines per element, IDS, MASK <f>.
    Frozen choice: one integer per line in IDS and MASK sections."""
    xyz = np.asarray(xyz)
    E, nq = xyz.shape[1], xyz.shape[2]
    with open(path, "w") as f:
        f.write(f"HEXMESH v1 {E} {nq - 1}\n")
        pts = xyz.reshape(3, -1).T
        for p in pts:
            f.write(f"{float(p[0])!r} {float(p[1])!r} {float(p[2])!r}\n")
        f.write("IDS\n")
        f.write("\n".join(str(int(v)) for v in np.asarray(ids).ravel()))
        f.write("\n")
        for name, mk in (masks or {}).items():
            f.write(f"MASK {name}\n")
            f.write("\n".join(str(int(v)) for v in np.asarray(mk).ravel()))
            f.write("\n")


def read_hexmesh(path):
    with open(path) as f:
        head = f.readline().split()
        if len(head) != 4 or head[0] != "HEXMESH" or head[1] != "v1":
            raise ValueError("not a HEXMESH v1 file")
        E, N = int(head[2]), int(head[3])
        nq = N + 1
        n = E * nq ** 3
        pts = np.array([[float(t) for t in f.readline().split()] for _ in range(n)])
        xyz = pts.T.reshape(3, E, nq, nq, nq)
        ids = None
        masks = {}
        line = f.readline()
        while line:
            tok = line.split()
            if not tok:
                line = f.readline()
                continue
            if tok[0] == "IDS":
                ids = np.array([int(f.readline()) for _ in range(n)], dtype=np.int64)
            elif tok[0] == "MASK":
                masks[tok[1]] = np.array([int(f.readline()) for _ in range(n)], dtype=np.int64)
            else:
                raise ValueError(f"unexpected section {tok[0]!r}")
            line = f.readline()
    return E, N, xyz, ids, masks
