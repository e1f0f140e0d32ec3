"""Meshes for the hot path: box generation, geometric factors, ids, masks,
HEXMESH v1 I/O -- the drop-in for ``nekmini.mesh``.

Geometry is produced ON DEVICE by libnekb200 (nk_box_coords,
nk_geom_factors, nk_box_ids, nk_box_mask) and kept resident in HBM in the
layouts the BK5 kernel streams:

    G    float64 [E][6][(N+1)^3]   (G11 G12 G13 G22 G23 G33)
    B    float64 [E][(N+1)^3]      (rho * J)
    ids  int64   [E*(N+1)^3]       (full global numbering, 1-based)
    mask uint8   [E][(N+1)^3]      (0 on Dirichlet points)

Frozen spec decisions (same as the oracle): element
order e = ex + nx*(ey + ny*ez); box ids = rank of the UNDEFORMED lattice point
in (z, y, x) order; 'sine' deformation
    x' = x + a Lx sin(2 pi X) sin(pi Y) sin(pi Z)   (and cyclic for y', z').
"""

import numpy as np

from . import _lib
from ._lib import ContractError, check, lib, ptr, stream_ptr
from .basis import SpectralBasis

FACES = ("x-", "x+", "y-", "y+", "z-", "z+")
DEFORM_CODES = {None: 0, "none": 0, "sine": 1}

__all__ = ["Mesh", "build_box_mesh", "geometric_factors", "assign_global_ids",
           "mesh_from_coords", "read_hexmesh", "write_hexmesh", "InvertedElementError",
           "DegenerateElementError", "normalize_bc", "singleton_ids"]


class InvertedElementError(ValueError):
    """Non-positive Jacobian after deformation."""


class DegenerateElementError(ValueError):
    """|J| < 1e-14."""


def normalize_bc(bc):
    """'dirichlet' | 'neumann' | 'periodic' for all faces, a dict face->kind or
    a 6-sequence in (x-, x+, y-, y+, z-, z+) order."""
    if isinstance(bc, str):
        out = dict.fromkeys(FACES, bc)
    elif isinstance(bc, dict):
        out = {f: bc.get(f, "neumann") for f in FACES}
    else:
        out = dict(zip(FACES, list(bc)))
    for f, kind in out.items():
        if kind not in ("dirichlet", "neumann", "periodic"):
            raise ValueError(f"unknown boundary kind {kind!r} on face {f}")
    for a in range(3):
        if (out[FACES[2 * a]] == "periodic") != (out[FACES[2 * a + 1]] == "periodic"):
            raise ValueError(f"periodic faces must come in pairs (axis {a})")
    return out


class Mesh:
    """Device-resident hex mesh (the SPEC Mesh type).

    ``E`` counts the elements held on this rank; ``elements`` (int64, or None
    for all) maps them to global element indices, ``rank_of_element`` is the
    partition when the mesh was built for a rank."""

    def __init__(self, N, E, G, B, ids, mask, basis, device, J=None, xyz=None, rx=None,
                 counts=None, extent=None, origin=None, bc=None, deformation=None,
                 elements=None):
        self.N, self.nq, self.E = N, N + 1, E
        self.G, self.B, self.ids, self.mask = G, B, ids, mask
        self.J, self.xyz, self.rx = J, xyz, rx
        self.basis, self.device = basis, device
        self.counts, self.extent, self.origin = counts, extent, origin
        self.bc, self.deformation, self.elements = bc, deformation, elements
        self.rank_of_element = None

    @property
    def order(self):
        return self.N

    @property
    def n_local(self):
        return self.E * self.nq ** 3

    def field_shape(self, ncomp=1):
        s = (self.E, self.nq, self.nq, self.nq)
        return s if ncomp == 1 else (ncomp,) + s

    def new_field(self, ncomp=1):
        import torch
        return torch.zeros(self.field_shape(ncomp), dtype=torch.float64, device=self.device)

    def element_centroids(self):
        """Centroids of the undeformed box elements (for RCB), (E, 3) host."""
        nx, ny, nz = self.counts
        el = np.arange(nx * ny * nz) if self.elements is None else np.asarray(self.elements)
        ex, ey, ez = el % nx, (el // nx) % ny, el // (nx * ny)
        h = np.array(self.extent) / np.array(self.counts)
        return np.stack([(ex + 0.5) * h[0], (ey + 0.5) * h[1], (ez + 0.5) * h[2]], axis=1) + \
            np.asarray(self.origin)


def _deform_spec(deformation):
    if deformation is None:
        return 0, 0.0
    if isinstance(deformation, str):
        return DEFORM_CODES[deformation], 0.05
    kind, amp = deformation
    if kind not in DEFORM_CODES:
        raise ValueError(f"unknown deformation {kind!r}")
    return DEFORM_CODES[kind], float(amp)


def _geom_from_xyz(N, E, xyz, basis, device, want_J=False, want_rx=False):
    import torch
    D, _, w = basis.device_arrays(device)
    nq3 = (N + 1) ** 3
    G = torch.empty((E, 6, N + 1, N + 1, N + 1), dtype=torch.float64, device=device)
    B = torch.empty((E, N + 1, N + 1, N + 1), dtype=torch.float64, device=device)
    J = torch.empty_like(B) if want_J else None
    rx = torch.empty((3, 3, E, N + 1, N + 1, N + 1), dtype=torch.float64, device=device) \
        if want_rx else None
    status = torch.full((2,), np.iinfo(np.int64).max, dtype=torch.int64, device=device)
    check(lib().nk_geom_factors(N, E, ptr(D), ptr(w), ptr(xyz), ptr(G), ptr(B), ptr(J), ptr(rx),
                                ptr(status), stream_ptr()), "geom_factors")
    st = status.cpu().numpy()
    if st[0] != np.iinfo(np.int64).max:
        raise DegenerateElementError(f"degenerate element {int(st[0])}: |J| < 1e-14")
    if st[1] != np.iinfo(np.int64).max:
        raise InvertedElementError(f"inverted element {int(st[1])}: J <= 0")
    del nq3
    return G, B, J, rx


def build_box_mesh(extent, counts, N, bc="dirichlet", deformation=None, origin=(0.0, 0.0, 0.0),
                   elements=None, device="cuda", keep_coords=False, keep_jacobian=False):
    """Box mesh built on device.

    deformation: None, 'sine', ('sine', amplitude) or a callable
    (x, y, z) -> (x', y', z') applied on host numpy arrays.
    elements: optional global element indices to build (a rank's share)."""
    import torch
    counts = tuple(int(c) for c in counts)
    if min(counts) < 1:
        raise ValueError("counts must be >= 1 in every direction")
    if isinstance(N, bool) or not isinstance(N, (int, np.integer)) or N < 1:
        from .basis import InvalidOrderError
        raise InvalidOrderError(f"polynomial order must be an integer >= 1, got {N!r}")
    bcn = normalize_bc(bc)
    basis = SpectralBasis.get(int(N))
    _, nodes, _ = basis.device_arrays(device)
    Etot = counts[0] * counts[1] * counts[2]
    if elements is None:
        eidx = None
        E = Etot
    else:
        eidx = torch.as_tensor(np.asarray(elements, dtype=np.int64), device=device)
        E = int(eidx.numel())
    nq = N + 1
    c32 = np.array(counts, dtype=np.int32)
    ext = np.array(extent, dtype=np.float64)
    org = np.array(origin, dtype=np.float64)
    callable_def = callable(deformation)
    kind, amp = (0, 0.0) if callable_def else _deform_spec(deformation)
    xyz = torch.empty((3, E, nq, nq, nq), dtype=torch.float64, device=device)
    s = stream_ptr()
    L = lib()
    check(L.nk_box_coords(N, E, ptr(eidx), ptr(c32), ptr(ext), ptr(org), kind, amp, ptr(nodes),
                          ptr(xyz), s), "box_coords")
    if callable_def:
        h = xyz.cpu().numpy()
        x, y, z = deformation(h[0], h[1], h[2])
        xyz = torch.as_tensor(np.stack([x, y, z]).astype(np.float64), device=device)
    G, B, J, _ = _geom_from_xyz(N, E, xyz, basis, device, want_J=keep_jacobian)
    ids = torch.empty(E * nq ** 3, dtype=torch.int64, device=device)
    per = np.array([bcn[FACES[2 * a]] == "periodic" for a in range(3)], dtype=np.int32)
    check(L.nk_box_ids(N, E, ptr(eidx), ptr(c32), ptr(per), ptr(ids), s), "box_ids")
    dir_ = np.array([bcn[f] == "dirichlet" for f in FACES], dtype=np.int32)
    mask = torch.empty((E, nq, nq, nq), dtype=torch.uint8, device=device)
    check(L.nk_box_mask(N, E, ptr(eidx), ptr(c32), ptr(dir_), ptr(mask), s), "box_mask")
    m = Mesh(N, E, G, B, ids, mask, basis, device, J=J, xyz=xyz if keep_coords else None,
             counts=counts, extent=tuple(float(v) for v in extent),
             origin=tuple(float(v) for v in origin), bc=bcn, deformation=deformation,
             elements=None if elements is None else np.asarray(elements, dtype=np.int64))
    return m


def mesh_coordinates(m):
    """GLL point coordinates (3, E, nq, nq, nq) of a mesh on its device: the
    stored ones, or (box meshes built without keep_coords) regenerated by
    nk_box_coords with the mesh's own counts / extent / deformation."""
    import torch
    if m.xyz is not None:
        return m.xyz
    if m.counts is None:
        raise ContractError("mesh has neither coordinates nor a box description")
    N, nq = m.N, m.nq
    _, nodes, _ = m.basis.device_arrays(m.device)
    eidx = None if m.elements is None else torch.as_tensor(m.elements, device=m.device)
    callable_def = callable(m.deformation)
    kind, amp = (0, 0.0) if callable_def else _deform_spec(m.deformation)
    xyz = torch.empty((3, m.E, nq, nq, nq), dtype=torch.float64, device=m.device)
    # host arrays bound to names: they must outlive the call
    c32 = np.array(m.counts, dtype=np.int32)
    ext = np.array(m.extent, dtype=np.float64)
    org = np.array(m.origin, dtype=np.float64)
    check(lib().nk_box_coords(N, m.E, ptr(eidx), ptr(c32), ptr(ext), ptr(org), kind, amp,
                              ptr(nodes), ptr(xyz), stream_ptr()), "box_coords")
    if callable_def:
        h = xyz.cpu().numpy()
        x, y, z = m.deformation(h[0], h[1], h[2])
        xyz = torch.as_tensor(np.stack([x, y, z]).astype(np.float64), device=m.device)
    return xyz


def geometric_factors(element_xyz, basis, device="cuda"):
    """(J, metrics, G, B) of one or more elements.

    element_xyz: (3, nq, nq, nq) or (3, E, nq, nq, nq) coordinates (numpy or
    tensor).  Computed on device; returned as numpy arrays with metrics
    rx[q][p] = dr_q/dx_p shaped (3, 3, [E,] nq, nq, nq)."""
    import torch
    x = torch.as_tensor(np.asarray(element_xyz.cpu() if hasattr(element_xyz, "cpu")
                                   else element_xyz, dtype=np.float64))
    single = x.dim() == 4
    if single:
        x = x.unsqueeze(1)
    E = x.shape[1]
    x = x.to(device).contiguous()
    G, B, J, rx = _geom_from_xyz(basis.order, E, x, basis, device, want_J=True, want_rx=True)
    out = [J.cpu().numpy(), rx.cpu().numpy(), G.cpu().numpy(), B.cpu().numpy()]
    if single:
        out = [out[0][0], out[1][:, :, 0], out[2][0], out[3][0]]
    return tuple(out)


def assign_global_ids(coords, tol_rel=1e-10):
    """Global ids from coordinates: snap to
    tol_rel x domain diameter, number unique points 1.. in (z, y, x) order.
    coords: (3, n) or (3, E, nq, nq, nq).  Host setup."""
    c = np.asarray(coords, dtype=np.float64).reshape(3, -1)
    lo = c.min(axis=1, keepdims=True)
    span = c.max(axis=1, keepdims=True) - lo
    h = tol_rel * max(float(np.sqrt((span ** 2).sum())), 1e-300)
    key = np.rint((c - lo) / h).astype(np.int64)
    order = np.lexsort(key)                       # last row (z) is the primary key
    k = key[:, order]
    start = np.empty(k.shape[1], dtype=bool)
    start[:1] = True
    start[1:] = np.any(k[:, 1:] != k[:, :-1], axis=0)
    ids = np.empty(k.shape[1], dtype=np.int64)
    ids[order] = np.cumsum(start)
    return ids


def singleton_ids(ids):
    """Ids held exactly once set to 0."""
    a = np.asarray(ids.cpu() if hasattr(ids, "cpu") else ids).ravel()
    _, inv, cnt = np.unique(a, return_inverse=True, return_counts=True)
    out = a.copy()
    out[(cnt[inv] == 1) | (a == 0)] = 0
    return out


def mesh_from_coords(xyz, N, ids=None, mask=None, device="cuda"):
    """Mesh from explicit GLL coordinates (e.g. a HEXMESH file)."""
    import torch
    basis = SpectralBasis.get(int(N))
    x = torch.as_tensor(np.ascontiguousarray(xyz, dtype=np.float64), device=device)
    E = x.shape[1]
    nq = N + 1
    G, B, J, _ = _geom_from_xyz(N, E, x, basis, device, want_J=True)
    if ids is None:
        ids = assign_global_ids(np.asarray(xyz))
    ids_t = torch.as_tensor(np.asarray(ids, dtype=np.int64), device=device)
    if mask is None:
        mask_t = torch.ones((E, nq, nq, nq), dtype=torch.uint8, device=device)
    else:
        mask_t = torch.as_tensor(np.asarray(mask, dtype=np.uint8).reshape(E, nq, nq, nq),
                                 device=device)
    return Mesh(N, E, G, B, ids_t, mask_t, basis, device, J=J, xyz=x)


# ------------------------------------------------------------ HEXMESH v1
# SPEC.md:161-162.  Frozen choices: one integer per line in IDS and MASK.

def write_hexmesh(path, xyz, ids, masks=None):
    xyz = np.asarray(xyz.cpu() if hasattr(xyz, "cpu") else xyz, dtype=np.float64)
    E, nq = xyz.shape[1], xyz.shape[2]
    pts = xyz.reshape(3, -1).T
    lines = [f"HEXMESH v1 {E} {nq - 1}"]
    lines += [f"{float(a)!r} {float(b)!r} {float(c)!r}" for a, b, c in pts]
    lines.append("IDS")
    lines += [str(int(v)) for v in np.asarray(ids.cpu() if hasattr(ids, "cpu") else ids).ravel()]
    for name, mk in (masks or {}).items():
        lines.append(f"MASK {name}")
        mk = mk.cpu() if hasattr(mk, "cpu") else mk
        lines += [str(int(v)) for v in np.asarray(mk).ravel()]
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def read_hexmesh(path):
    """Returns (E, N, xyz (3,E,nq,nq,nq), ids or None, {field: mask})."""
    with open(path) as f:
        tokens = f.read().split("\n")
    it = iter(tokens)
    head = next(it).split()
    if len(head) != 4 or head[:2] != ["HEXMESH", "v1"]:
        raise ValueError(f"{path}: not a HEXMESH v1 file")
    E, N = int(head[2]), int(head[3])
    nq = N + 1
    n = E * nq ** 3
    pts = np.array([next(it).split() for _ in range(n)], dtype=np.float64)
    xyz = np.ascontiguousarray(pts.T.reshape(3, E, nq, nq, nq))
    ids, masks = None, {}
    for line in it:
        t = line.split()
        if not t:
            continue
        if t[0] == "IDS":
            ids = np.array([next(it) for _ in range(n)], dtype=np.int64)
        elif t[0] == "MASK" and len(t) == 2:
            masks[t[1]] = np.array([next(it) for _ in range(n)], dtype=np.int64)
        else:
            raise ValueError(f"{path}: unexpected section {line!r}")
    return E, N, xyz, ids, masks
