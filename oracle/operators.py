"""Oracle: element-local operators (BK5 stiffness, mass, Jacobi diagonal).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  * apply_stiffness_local  SPEC.md:370-378; PAPER.md:1150-1162 (tensor
    contractions), PAPER.md:1240-1266 (w = D^T G D u with six G factors).
  * apply_mass / inner_product  SPEC.md:380-388.
  * Helmholtz  H = lam0 A + lam1 B.
  * extract_diagonal  SPEC.md:400-408 (closed form from D-hat and G, then
    assembled by gs(+)).
  * dense_element_stiffness: Eq. (25) entries A_ab = sum_q rho_q J_q
    grad(phi_a).grad(phi_b) evaluated directly with metrics -- the independent
    dense oracle of SPEC.md:377, 407, 431.
  * KernelCounters formulas SPEC.md:363, 373 (12(N+1)^4 + 15(N+1)^3 flops per
    element; 7(N+1)^3 memory refs per element).

Layout: u, w (E, nq, nq, nq) indexed [e][k][j][i]; G (E, 6, nq, nq, nq).
"""

import numpy as np


def bk5(D, G, u, lam0=1.0, B=None, lam1=0.0):
    """w = lam0 * A_L u + lam1 * B u (element-local, unassembled)."""
    D = np.asarray(D, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    E, nq = u.shape[0], u.shape[1]
    DT = D.T
    # forward derivatives (r along i, s along j, t along k)
    ur = u @ DT                                          # sum_m D[i,m] u[k,j,m]
    us = np.matmul(D, u)                                 # sum_m D[j,m] u[k,m,i]
    ut = np.matmul(D, u.reshape(E, nq, nq * nq)).reshape(u.shape)  # sum_m D[k,m] u[m,j,i]
    g = G
    gr = g[:, 0] * ur + g[:, 1] * us + g[:, 2] * ut
    gs = g[:, 1] * ur + g[:, 3] * us + g[:, 4] * ut
    gt = g[:, 2] * ur + g[:, 4] * us + g[:, 5] * ut
    w = gr @ D                                           # sum_m D[m,i] gr[k,j,m]
    w += np.matmul(DT, gs)                               # sum_m D[m,j] gs[k,m,i]
    w += np.matmul(DT, gt.reshape(E, nq, nq * nq)).reshape(u.shape)
    if lam0 != 1.0:
        w *= lam0
    if B is not None and lam1 != 0.0:
        w += lam1 * B * u
    return w


def bk5_flops(N, E):
    nq = N + 1
    return E * (12 * nq ** 4 + 15 * nq ** 3)


def bk5_memrefs(N, E):
    return 7 * E * (N + 1) ** 3


def apply_mass(B, u):
    return np.asarray(B) * np.asarray(u)


def inner_product(B, v, u):
    """(v, u)_B = sum over local points of v B u.  Local
    points, no multiplicity weighting: B is the unassembled local mass, so the
    local sum equals the assembled integral for continuous v, u."""
    return float(np.sum(np.asarray(v) * np.asarray(B) * np.asarray(u)))


def local_diagonal(D, G, lam0=1.0, B=None, lam1=0.0):
    """Closed-form diag(A^e) per element:
    diag[k,j,i] = sum_m D[m,i]^2 G11[k,j,m] + sum_m D[m,j]^2 G22[k,m,i]
                + sum_m D[m,k]^2 G33[m,j,i] + 2 D[i,i] D[j,j] G12[k,j,i]
                + 2 D[i,i] D[k,k] G13[k,j,i] + 2 D[j,j] D[k,k] G23[k,j,i]."""
    D = np.asarray(D, dtype=np.float64)
    E, nq = G.shape[0], G.shape[2]
    D2 = D * D
    d = np.diag(D)
    g = G
    out = g[:, 0] @ D2                                   # sum_m D[m,i]^2 G11[k,j,m]
    out += np.matmul(D2.T, g[:, 3])                      # sum_m D[m,j]^2 G22[k,m,i]
    out += np.matmul(D2.T, g[:, 5].reshape(E, nq, nq * nq)).reshape(out.shape)
    di = d[None, None, None, :]
    dj = d[None, None, :, None]
    dk = d[None, :, None, None]
    out += 2 * di * dj * g[:, 1] + 2 * di * dk * g[:, 2] + 2 * dj * dk * g[:, 4]
    out *= lam0
    if B is not None and lam1 != 0.0:
        out += lam1 * B
    return out


def dense_element_stiffness(D, rx, J, w):
    """Dense A^e from Eq. (25) by quadrature with explicit metrics.

    rx: (3,3,nq,nq,nq) metrics dr_q/dx_p for ONE element; J: (nq,nq,nq).
    Returns (nq^3, nq^3) matrix in [k][j][i] flattened order."""
    nq = D.shape[0]
    I = np.eye(nq)
    # dphi_b/dr_q at quadrature point a (flattened k,j,i order: i fastest)
    Dr = np.kron(I, np.kron(I, D))
    Ds = np.kron(I, np.kron(D, I))
    Dt = np.kron(D, np.kron(I, I))
    dref = [Dr, Ds, Dt]
    rho = (w[:, None, None] * w[None, :, None] * w[None, None, :]).ravel()
    wq = rho * J.ravel()
    A = np.zeros((nq ** 3, nq ** 3))
    for p in range(3):  # physical direction x_p
        gx = sum(rx[q, p].ravel()[:, None] * dref[q] for q in range(3))  # (quad, basis)
        A += gx.T @ (wq[:, None] * gx)
    return A


def dense_assembled(ids, A_blocks, lam1=0.0, B=None):
    """Q^T blockdiag(A^e) Q with Q from ids (ids must be the full numbering)."""
    from .gs import dense_Q
    n = sum(a.shape[0] for a in A_blocks)
    AL = np.zeros((n, n))
    o = 0
    for a in A_blocks:
        m = a.shape[0]
        AL[o:o + m, o:o + m] = a
        o += m
    if B is not None and lam1:
        AL += lam1 * np.diag(np.ravel(B))
    Q = dense_Q(ids)
    return Q, Q.T @ AL @ Q, AL
