"""GLL basis (host setup): the drop-in for ``nekmini.basis``.

Same public names and semantics as /root/reference/pkg/src/nekmini/basis.py
(``SpectralBasis``/``.get``/``.n``, ``gll_rule``, ``interp_matrix``,
``InvalidOrderError``; basis.py:11-189).  Setup-time only: the arrays are
computed once in float64 on the host, frozen, and uploaded to the device
unchanged (``SpectralBasis.device_arrays``) -- the BK5 kernels never
re-derive D-hat.  Bit-for-bit equal to the reference (tests/golden).
"""

import numpy as np

__all__ = ["SpectralBasis", "gll_rule", "interp_matrix", "InvalidOrderError", "InterpMatrix",
           "diff_matrix", "lagrange_interp_matrix"]


class InvalidOrderError(ValueError):
    """Order outside the supported range (reference basis.py:14)."""


def _legendre_triple(n, x):
    """P_n(x), P_n'(x), P_n''(x) via Bonnet's recurrence (basis.py:18-38)."""
    x = np.asarray(x, dtype=np.float64)
    one, zero = np.ones_like(x), np.zeros_like(x)
    if n == 0:
        return one, zero, zero.copy()
    prev = (one, zero, zero.copy())
    cur = (x.copy(), one.copy(), zero.copy())
    for k in range(2, n + 1):
        a, b = (2.0 * k - 1.0) / k, (k - 1.0) / k
        p1, d1, s1 = cur
        p0, d0, s0 = prev
        nxt = (a * x * p1 - b * p0,
               a * (p1 + x * d1) - b * d0,
               a * (2.0 * d1 + x * s1) - b * s0)
        prev, cur = cur, nxt
    return cur


def gll_rule(N):
    """(nodes, weights) of the (N+1)-point GLL rule (basis.py:41-69)."""
    if isinstance(N, bool) or not isinstance(N, (int, np.integer)) or N < 1:
        raise InvalidOrderError(f"polynomial order must be an integer >= 1, got {N!r}")
    N = int(N)
    xi = -np.cos(np.pi * np.arange(N + 1) / N)
    for _it in range(100):
        _, dP, d2P = _legendre_triple(N, xi)
        g = (1.0 - xi * xi) * dP                     # roots: GLL nodes
        dg = -2.0 * xi * dP + (1.0 - xi * xi) * d2P
        g[[0, -1]] = 0.0
        dg[[0, -1]] = 1.0
        delta = g / dg
        xi -= delta
        if np.max(np.abs(delta)) < 1e-15:
            break
    xi[0], xi[-1] = -1.0, 1.0
    xi = 0.5 * (xi - xi[::-1])
    PN = _legendre_triple(N, xi)[0]
    rho = 2.0 / (N * (N + 1) * PN * PN)
    rho = 0.5 * (rho + rho[::-1])
    return xi, rho


def _bary(nodes):
    diffs = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diffs, 1.0)
    return 1.0 / np.prod(diffs, axis=1)


def diff_matrix(nodes):
    """D[a, i] = h_i'(nodes[a]); zero row sums by construction (basis.py:80-96)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    lam = _bary(nodes)
    with np.errstate(divide="ignore", invalid="ignore"):
        D = (lam[None, :] / lam[:, None]) / (nodes[:, None] - nodes[None, :])
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, -D.sum(axis=1))
    return D


def lagrange_interp_matrix(from_nodes, to_nodes):
    """J[a, i] = h_i(to_nodes[a]), second barycentric form (basis.py:99-117)."""
    src = np.asarray(from_nodes, dtype=np.float64)
    dst = np.asarray(to_nodes, dtype=np.float64)
    lam = _bary(src)
    d = dst[:, None] - src[None, :]
    hit = np.abs(d) < 1e-14
    with np.errstate(divide="ignore", invalid="ignore"):
        t = lam[None, :] / d
        J = t / np.sum(t, axis=1, keepdims=True)
    rows = hit.any(axis=1)
    J[rows] = 0.0
    J[rows, np.argmax(hit[rows], axis=1)] = 1.0
    return J


class SpectralBasis:
    """Immutable GLL nodes, weights and D-hat for one order (basis.py:120-156)."""

    _cache = {}

    def __init__(self, order):
        nodes, weights = gll_rule(order)
        self.order = int(order)
        self.nodes = nodes
        self.weights = weights
        self.diff = diff_matrix(nodes)
        for a in (self.nodes, self.weights, self.diff):
            a.flags.writeable = False
        self._dev = {}

    @property
    def n(self):
        return self.order + 1

    def __repr__(self):
        return f"SpectralBasis(order={self.order})"

    @classmethod
    def get(cls, order):
        b = cls._cache.get(order)
        if b is None:
            b = cls._cache[order] = cls(order)
        return b

    def device_arrays(self, device="cuda"):
        """(D, nodes, weights) as float64 device tensors (uploaded once)."""
        import torch
        key = str(device)
        if key not in self._dev:
            mk = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=device)
            self._dev[key] = (mk(self.diff), mk(self.nodes), mk(self.weights))
        return self._dev[key]


class InterpMatrix:
    """Interpolation operator between node sets (basis.py:159-173)."""

    def __init__(self, from_order, to_order, values):
        self.from_order = from_order
        self.to_order = to_order
        self.values = values

    def __repr__(self):
        return f"InterpMatrix({self.from_order} -> {self.to_order})"


def interp_matrix(from_basis, to_nodes, to_order=None):
    """basis.py:176-189: to_nodes may be a SpectralBasis or an array."""
    if isinstance(to_nodes, SpectralBasis):
        to_order, to_nodes = to_nodes.order, to_nodes.nodes
    to_nodes = np.asarray(to_nodes, dtype=np.float64)
    if to_order is None:
        to_order = len(to_nodes) - 1
    return InterpMatrix(from_basis.order, to_order,
                        lagrange_interp_matrix(from_basis.nodes, to_nodes))
