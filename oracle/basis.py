"""Oracle: 1-D Gauss-Lobatto-Legendre rule and differentiation matrix.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates /root/reference/pkg/src/nekmini/basis.py:
  * Legendre three-term recurrence for P, P', P''      -> basis.py:18-38
  * Newton on (1-r^2) P'_N from Chebyshev-Lobatto guesses,
    |dx| < 1e-15 stop, symmetrisation of nodes/weights  -> basis.py:41-69
  * barycentric weights                                 -> basis.py:72-77
  * D[a,i] = h_i'(xi_a), diagonal = -(off-diagonal row sum) -> basis.py:80-96
  * Lagrange interpolation (second barycentric form)    -> basis.py:99-117
Pinned bit-for-bit against tests/golden/basis_ref.npz (generated from the
reference module by tests/golden/make_golden.py).
"""

import numpy as np


class InvalidOrderError(ValueError):
    """Polynomial order outside the supported range (basis.py:14)."""


def legendre_with_derivs(n, x):
    """(P_n, P_n', P_n'') at x by the Bonnet recurrence (basis.py:18-38)."""
    x = np.asarray(x, dtype=np.float64)
    if n == 0:
        return np.ones_like(x), np.zeros_like(x), np.zeros_like(x)
    pm, dm, sm = np.ones_like(x), np.zeros_like(x), np.zeros_like(x)
    p, d, s = x.copy(), np.ones_like(x), np.zeros_like(x)
    for k in range(2, n + 1):
        c1 = (2.0 * k - 1.0) / k
        c0 = (k - 1.0) / k
        pn = c1 * x * p - c0 * pm
        dn = c1 * (p + x * d) - c0 * dm
        sn = c1 * (2.0 * d + x * s) - c0 * sm
        pm, dm, sm = p, d, s
        p, d, s = pn, dn, sn
    return p, d, s


def gll_rule(N):
    """GLL nodes and weights for order N (basis.py:41-69)."""
    if not isinstance(N, (int, np.integer)) or isinstance(N, bool) or N < 1:
        raise InvalidOrderError(f"order must be an integer >= 1, got {N!r}")
    N = int(N)
    r = -np.cos(np.pi * np.arange(N + 1) / N)
    for _ in range(100):
        _, dp, ddp = legendre_with_derivs(N, r)
        f = (1.0 - r * r) * dp
        fp = -2.0 * r * dp + (1.0 - r * r) * ddp
        f[0] = f[-1] = 0.0
        fp[0] = fp[-1] = 1.0
        step = f / fp
        r -= step
        if np.max(np.abs(step)) < 1e-15:
            break
    r[0], r[-1] = -1.0, 1.0
    r = 0.5 * (r - r[::-1])
    pN, _, _ = legendre_with_derivs(N, r)
    w = 2.0 / (N * (N + 1) * pN * pN)
    w = 0.5 * (w + w[::-1])
    return r, w


def barycentric_weights(nodes):
    n = len(nodes)
    out = np.ones(n)
    for a in range(n):
        out[a] = 1.0 / np.prod(nodes[a] - np.delete(nodes, a))
    return out


def diff_matrix(nodes):
    """D[a, i] = h_i'(nodes[a]); rows sum to zero exactly (basis.py:80-96)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    n = len(nodes)
    lam = barycentric_weights(nodes)
    D = np.zeros((n, n))
    for a in range(n):
        for i in range(n):
            if i != a:
                D[a, i] = (lam[i] / lam[a]) / (nodes[a] - nodes[i])
        D[a, a] = -np.sum(D[a, :])
    return D


def interp_matrix(from_nodes, to_nodes):
    """J[a, i] = h_i(to_nodes[a]) (basis.py:99-117)."""
    from_nodes = np.asarray(from_nodes, dtype=np.float64)
    to_nodes = np.asarray(to_nodes, dtype=np.float64)
    lam = barycentric_weights(from_nodes)
    J = np.zeros((len(to_nodes), len(from_nodes)))
    for a, y in enumerate(to_nodes):
        diff = y - from_nodes
        hit = np.abs(diff) < 1e-14
        if hit.any():
            J[a, int(np.argmax(hit))] = 1.0
        else:
            t = lam / diff
            J[a] = t / np.sum(t)
    return J


class Basis:
    """Nodes, weights and D-hat for one order (basis.py:120-156)."""

    _cache = {}

    def __init__(self, order):
        self.nodes, self.weights = gll_rule(order)
        self.order = int(order)
        self.diff = diff_matrix(self.nodes)

    @property
    def n(self):
        return self.order + 1

    @classmethod
    def get(cls, order):
        b = cls._cache.get(order)
        if b is None:
            b = cls._cache[order] = cls(order)
        return b
