"""GPU parity: the p-multigrid preconditioner (paper_2104_05829_b200.multigrid,
libnekb200 nk_interp3 / nk_cheb_step / nk_dense_matvec + BK5 + gs at every
order) against oracle/pmg.py.  Bars: lambda_max, smoother, coarse solve and
V-cycle within 1e-10 relative L2 (FP64, different summation order); PCG
iterations within +-1 of the oracle at the same tolerance."""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import pmg as opmg
from oracle import solvers as osol

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import multigrid as mg  # noqa: E402

TOL = 1e-10


def rel_l2(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def pair(counts, N, deformation=("sine", 0.05), bc="dirichlet", lam0=1.0, lam1=0.0):
    m = nk.build_box_mesh((1, 1, 1), counts, N, bc=bc, deformation=deformation)
    op = nk.PoissonOperator(m, lam0=lam0, lam1=lam1)
    h = nk.MultigridHierarchy(op)
    o = opmg.build_hierarchy((1, 1, 1), counts, N, bc=bc, deformation=deformation,
                             lam0=lam0, lam1=lam1)
    return op, h, o


def rand_assembled(lv, seed):
    x = np.random.default_rng(seed).standard_normal(lv.mask.size)
    return lv.mask * ogs.gs_op(lv.mesh.ids, lv.wt * x)


def rhs(lv):
    X = lv.mesh.xyz.reshape(3, -1)
    f = 3 * np.pi ** 2 * np.prod(np.sin(np.pi * X), axis=0)
    return lv.mask * ogs.gs_op(lv.mesh.ids, lv.mesh.B.ravel() * f)


@pytest.mark.parametrize("N,counts", [(2, (2, 2, 2)), (3, (3, 2, 2)), (5, (2, 2, 2)),
                                      (7, (2, 2, 2)), (8, (2, 2, 1)), (12, (1, 2, 1))])
def test_hierarchy_lambda_and_vcycle(N, counts):
    op, h, o = pair(counts, N)
    assert h.orders == opmg.orders_for(N)
    for lg, lo in zip(h.levels[:-1], o["levels"][:-1]):
        assert abs(lg.lmax - lo.lmax) < 1e-10 * lo.lmax
        assert rel_l2(lg.invD.cpu().numpy(), lo.invD) < 1e-13
    r = rand_assembled(o["levels"][0], 11)
    z = nk.pmg_preconditioner(h, dev(r)).cpu().numpy()
    zo = opmg.vcycle(o, r)
    assert rel_l2(z, zo) < TOL


@pytest.mark.parametrize("level", [0, 1])
def test_chebyshev_smooth_matches_oracle(level):
    op, h, o = pair((2, 2, 2), 7)
    lo = o["levels"][level]
    r = rand_assembled(lo, 3 + level)
    for deg in (1, 2, 3):
        e = nk.chebyshev_smooth(h, level, dev(r), degree=deg).cpu().numpy()
        eo = opmg.chebyshev_smooth(lo, r, deg, lo.lo, lo.hi)
        assert rel_l2(e, eo) < TOL


def test_coarse_solve_matches_oracle_and_unit_vector():
    op, h, o = pair((3, 2, 2), 3)
    lo = o["levels"][-1]
    r = rand_assembled(lo, 9)
    e = nk.coarse_solve(h, dev(r)).cpu().numpy()
    Q, Ainv = lo.coarse
    eo = lo.mask * (Q @ (Ainv @ (Q.T @ (lo.wt * r))))
    assert rel_l2(e, eo) < 1e-11
    # rhs = A e_k -> e_k
    ids = lo.mesh.ids
    k = ids[lo.mask.astype(bool)][3]
    ek = (ids == k).astype(np.float64)
    Aek = opmg._apply_op(lo, ek)
    z = nk.coarse_solve(h, dev(Aek)).cpu().numpy()
    assert np.max(np.abs(z - ek)) < 1e-12


def test_coarse_neumann_singular_pinned():
    op, h, o = pair((2, 2, 2), 3, bc="neumann", deformation=None)
    lo = o["levels"][-1]
    r = opmg._apply_op(lo, rand_assembled(lo, 2))
    e = nk.coarse_solve(h, dev(r)).cpu().numpy()
    Q, Ainv = lo.coarse
    eo = lo.mask * (Q @ (Ainv @ (Q.T @ (lo.wt * r))))
    assert rel_l2(e, eo) < 1e-10


def test_vcycle_zero_symmetric_and_helmholtz():
    op, h, o = pair((2, 2, 2), 5, lam0=0.5, lam1=20.0)
    lv = o["levels"][0]
    z0 = nk.pmg_preconditioner(h, torch.zeros(op.n, dtype=torch.float64, device="cuda"))
    assert not bool(z0.abs().max() > 0)
    r1, r2 = rand_assembled(lv, 5), rand_assembled(lv, 6)
    z1 = nk.pmg_preconditioner(h, dev(r1)).cpu().numpy()
    z2 = nk.pmg_preconditioner(h, dev(r2)).cpu().numpy()
    a, b = np.sum(lv.wt * z1 * r2), np.sum(lv.wt * r1 * z2)
    assert abs(a - b) < 1e-11 * abs(a)
    assert rel_l2(z1, opmg.vcycle(o, r1)) < TOL


@pytest.mark.parametrize("N,counts,deform", [(7, (2, 2, 2), ("sine", 0.05)),
                                             (7, (4, 4, 4), ("sine", 0.05)),
                                             (5, (3, 3, 3), None),
                                             (4, (3, 2, 2), ("sine", 0.05))])
def test_pmg_pcg_iterations_match_oracle(N, counts, deform):
    op, h, o = pair(counts, N, deformation=deform)
    lv = o["levels"][0]
    b = rhs(lv)
    A = opmg.fine_operator(o)
    ro = osol.pcg(A, lambda r: opmg.vcycle(o, r), b, tol=1e-8, max_iter=200, weights=lv.wt)
    s = nk.MultigridPCG(op, h, tol=1e-8, max_iter=200)
    res = s.solve(dev(b))
    assert res.converged and ro.converged
    assert abs(res.iterations - ro.iterations) <= 1
    x = res.x.cpu().numpy()
    assert np.max(np.abs(x - ro.x)) < 1e-7 * np.max(np.abs(ro.x))
    # strictly fewer iterations than Jacobi-PCG on the same problem
    rj = nk.pcg(op, nk.JacobiPreconditioner(op), dev(b), tol=1e-8, max_iter=3000)
    assert res.iterations < rj.iterations
    # solving again reuses the captured graph and reproduces the result bitwise
    res2 = s.solve(dev(b))
    assert res2.iterations == res.iterations
    assert torch.equal(res2.x, res.x) or np.array_equal(res2.x.cpu().numpy(), x)


def test_pmg_pcg_graph_equals_eager_and_pcg_dispatch():
    op, h, o = pair((3, 3, 3), 6)
    b = dev(rhs(o["levels"][0]))
    r1 = nk.MultigridPCG(op, h, tol=1e-9, max_iter=100, use_graph=True).solve(b)
    x1 = r1.x.clone()
    r2 = nk.MultigridPCG(op, h, tol=1e-9, max_iter=100, use_graph=False).solve(b)
    assert r1.iterations == r2.iterations
    assert torch.equal(x1, r2.x)
    r3 = nk.pcg(op, h, b, tol=1e-9, max_iter=100)          # routed to MultigridPCG
    assert r3.iterations == r1.iterations
    r4 = nk.pcg(op, h, b, tol=1e-9, max_iter=100, flexible=True)
    assert abs(r4.iterations - r1.iterations) <= 1


def test_coordinate_mesh_hierarchy_matches_box():
    """Explicit-coordinate meshes: coarse levels from interpolated
    coordinates.  On an affine box the interpolation is exact, so the
    V-cycle equals the box-mesh one."""
    mb = nk.build_box_mesh((1, 1, 1), (2, 3, 2), 5, keep_coords=True)
    mc = nk.mesh.mesh_from_coords(mb.xyz.cpu().numpy(), 5, ids=mb.ids.cpu().numpy(),
                                  mask=mb.mask.cpu().numpy())
    hb = nk.MultigridHierarchy(nk.PoissonOperator(mb))
    hc = nk.MultigridHierarchy(nk.PoissonOperator(mc))
    r = torch.randn(mb.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(hb.levels[0].op.gs, r)
    r *= mb.mask.reshape(-1).to(r.dtype)
    zb = nk.pmg_preconditioner(hb, r).cpu().numpy()
    zc = nk.pmg_preconditioner(hc, r).cpu().numpy()
    assert rel_l2(zc, zb) < 1e-9


def test_contract_errors():
    m = nk.build_box_mesh((1, 1, 1), (2, 2, 2), 3)
    op = nk.PoissonOperator(m)
    with pytest.raises(nk.ContractError):
        nk.MultigridHierarchy(op, degree=0)
    with pytest.raises(nk.ContractError):
        nk.MultigridHierarchy(op, bounds=(1.1, 0.1))
    with pytest.raises(nk.ContractError):
        nk.MultigridHierarchy(op, coarse="amg")
    h = nk.MultigridHierarchy(op)
    with pytest.raises(nk.ContractError):
        h.apply(torch.zeros(5, dtype=torch.float64, device="cuda"))
    with pytest.raises(nk.ContractError):
        nk.chebyshev_smooth(h, len(h.levels) - 1, torch.zeros(8, dtype=torch.float64,
                                                               device="cuda"))


def test_iterative_coarse_solve():
    """coarse='pcg': fused Jacobi-PCG on the order-1 level to coarse_tol --
    the scalable stand-in for the paper's AMG coarse solver.  Approximates the
    dense coarse solve to the inner tolerance; the flexible outer PCG needs at
    most a couple more iterations than with the exact coarse solve."""
    op, hd, o = pair((4, 4, 3), 7)
    hp = nk.MultigridHierarchy(op, coarse="pcg", coarse_tol=1e-6, coarse_iters=200)
    assert hp.levels[-1].cpcg is not None and hd.levels[-1].cpcg is None
    lo = o["levels"][-1]
    r = rand_assembled(lo, 9)
    ed = nk.coarse_solve(hd, dev(r)).cpu().numpy()
    ep = nk.coarse_solve(hp, dev(r)).cpu().numpy()
    assert rel_l2(ep, ed) < 1e-4
    b = dev(rhs(o["levels"][0]))
    rd = nk.MultigridPCG(op, hd, tol=1e-8, max_iter=200, flexible=True).solve(b)
    xd = rd.x.clone()
    sp = nk.MultigridPCG(op, nk.MultigridHierarchy(op, coarse="pcg"), tol=1e-8, max_iter=200)
    assert sp.flexible                      # auto: nonlinear preconditioner
    rp = sp.solve(b)
    assert rp.converged and rp.iterations <= rd.iterations + 3
    assert float((rp.x - xd).abs().max()) < 1e-6 * float(xd.abs().max())
    with pytest.raises(nk.ContractError):
        nk.MultigridHierarchy(op, coarse="amg")


@pytest.mark.parametrize("n", [1, 7, 64, 6859])
def test_dense_matvec32_matches_fp64(n):
    """nk_dense_matvec32 (the 32-bit smoothing mode's coarse inverse, FP32
    storage, FP64 sums; row pitch lda = n rounded up to 4, zero padded) vs the
    FP64 dense matvec: the FP32 rounding of A only (<= 1e-6 relative)."""
    from paper_2104_05829_b200._lib import check, lib, ptr
    L = lib()
    g = torch.Generator(device="cuda").manual_seed(n)
    A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    lda = (n + 3) // 4 * 4
    A32 = torch.zeros((n, lda), dtype=torch.float32, device="cuda")
    A32[:, :n] = A.float()
    x = torch.zeros(lda, dtype=torch.float64, device="cuda")
    x[:n] = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    y64 = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    check(L.nk_dense_matvec32(n, lda, ptr(A32), ptr(x), ptr(y), None, s), "dense_matvec32")
    check(L.nk_dense_matvec(n, ptr(A), ptr(x), ptr(y64), None, s), "dense_matvec")
    ref = A32[:, :n].double() @ x[:n]
    assert float(torch.linalg.norm(y - ref)) <= 1e-12 * float(torch.linalg.norm(ref))
    assert float(torch.linalg.norm(y - y64)) <= 1e-6 * float(torch.linalg.norm(y64))
    assert L.nk_dense_matvec32(n, lda + 1, ptr(A32), ptr(x), ptr(y), None, s) != 0
