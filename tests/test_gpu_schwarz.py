"""GPU parity: FDM local solves and overlapping Schwarz smoothers
(paper_2104_05829_b200.schwarz; libnekb200 nk_fdm / nk_schwarz_post + gs)
and the p-multigrid hierarchy with every SmootherConfig kind, against
oracle/schwarz.py and oracle/pmg.py.  Bars: FDM and Schwarz applications
within 1e-12 relative L2 (FP64, different summation order), lambda_max and
V-cycles within 1e-9, flexible-PCG iteration counts within +-1 of the
oracle at the same tolerance."""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om
from oracle import pmg as opmg
from oracle import schwarz as osz
from oracle import solvers as osol

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_05829_b200 as nk  # noqa: E402


def rel_l2(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def pair(counts, N, bc="dirichlet", deformation=("sine", 0.05), lam0=1.0, lam1=0.0):
    m = nk.build_box_mesh((1, 1, 1), counts, N, bc=bc, deformation=deformation)
    o = om.build_box_mesh((1, 1, 1), counts, N, bc=bc, deformation=deformation)
    op = nk.PoissonOperator(m, lam0=lam0, lam1=lam1)
    f = osz.fdm_setup(o.xyz, o.ids, o.mask, o.E, N, o.basis.diff, o.basis.weights, lam0, lam1)
    return m, o, op, f


def assembled_random(o, seed):
    x = np.random.default_rng(seed).standard_normal(o.mask.size)
    return o.mask.ravel() * ogs.gs_op(o.ids, x / ogs.multiplicity(o.ids))


CASES = [((3, 2, 2), 1, "dirichlet"), ((2, 2, 2), 2, "dirichlet"), ((3, 2, 2), 3, "dirichlet"),
         ((2, 3, 2), 5, "periodic"), ((2, 2, 2), 7, "dirichlet"), ((2, 1, 2), 7, "neumann"),
         ((2, 2, 1), 9, "dirichlet"), ((1, 2, 1), 12, "dirichlet"), ((1, 1, 2), 15, "dirichlet")]


@pytest.mark.parametrize("counts,N,bc", CASES)
def test_fdm_local_solve_matches_oracle(counts, N, bc):
    m, o, op, f = pair(counts, N, bc=bc, lam0=0.8, lam1=(0.0 if bc == "dirichlet" else 2.5))
    sm = nk.SchwarzSmoother(op, "asm")
    assert np.array_equal(sm.fmap.cpu().numpy(), f.fmap)
    r = assembled_random(o, N)
    u = nk.fdm_local_solve(sm, dev(r)).cpu().numpy()
    uo = osz.fdm_solve(f, osz.extend(f, r))
    # sampled (non-dropped) points only: outputs at never-sampled box points
    # are discarded by both smoothers
    used = f.ext_ids.reshape(u.shape) != 0
    assert rel_l2(u[used], uo[used]) < 1e-12
    assert not torch.any(nk.fdm_local_solve(sm, torch.zeros_like(dev(r))))


@pytest.mark.parametrize("counts,N,bc", [((3, 2, 2), 1, "dirichlet"), ((2, 3, 2), 5, "periodic"),
                                         ((3, 3, 3), 7, "dirichlet"), ((2, 1, 2), 7, "neumann"),
                                         ((2, 2, 1), 12, "dirichlet"), ((1, 2, 2), 13, "dirichlet")])
def test_fdm_tensor_core_path_matches_line_kernel(counts, N, bc):
    """NK_KNOB_FDM: the FP64 tensor-core FDM (mma.sync m8n8k4, N + 3 <= 16)
    against the CUDA-core line kernel on the same extended boxes -- the same
    algorithm with sums in a different order (1e-13), ASM and RAS outputs."""
    from paper_2104_05829_b200._lib import lib
    L = lib()
    m, o, op, f = pair(counts, N, bc=bc, lam0=0.8, lam1=(0.0 if bc == "dirichlet" else 2.5))
    r = dev(assembled_random(o, 7 + N))
    outs = {}
    try:
        for kn in (0, 1):
            L.nk_set_knob(3, kn)
            for kind in ("asm", "ras"):
                sm = nk.SchwarzSmoother(op, kind)
                outs[(kn, kind, "fdm")] = nk.fdm_local_solve(sm, r).cpu().numpy()
                z = torch.empty_like(r)
                sm.apply(r, z)
                outs[(kn, kind, "apply")] = z.cpu().numpy()
    finally:
        L.nk_set_knob(3, 2)
    for kind in ("asm", "ras"):
        for what in ("fdm", "apply"):
            a, b = outs[(1, kind, what)], outs[(0, kind, what)]
            assert rel_l2(a, b) < 1e-13, (kind, what)


@pytest.mark.parametrize("kind", ["asm", "ras"])
@pytest.mark.parametrize("counts,N,bc", CASES)
def test_schwarz_smooth_matches_oracle(kind, counts, N, bc):
    m, o, op, f = pair(counts, N, bc=bc)
    sm = nk.SchwarzSmoother(op, kind)
    r = assembled_random(o, 100 + N)
    z = nk.schwarz_smooth(sm, dev(r)).cpu().numpy()
    zo = osz.schwarz_smooth(f, kind, r, o.ids, o.mask)
    assert rel_l2(z, zo) < 1e-12
    if kind == "asm":
        assert rel_l2(sm.W.cpu().numpy(), f.Wext) < 1e-15
    # z is continuous: every copy of a shared point holds the same value
    zz = ogs.gs_op(o.ids, z) / ogs.multiplicity(o.ids)
    assert np.max(np.abs(zz - z)) <= 1e-14 * np.max(np.abs(z))


def test_single_element_asm_equals_ras_and_affine_exact_inverse():
    m, o, op, f = pair((1, 1, 1), 4, deformation=None)
    r = assembled_random(o, 1)
    za = nk.SchwarzSmoother(op, "asm")(dev(r))
    zr = nk.SchwarzSmoother(op, "ras")(dev(r))
    assert rel_l2(za.cpu().numpy(), zr.cpu().numpy()) < 1e-14
    # the surrogate of an affine element with Dirichlet faces is the element:
    # A z = r on the unmasked points
    Az = op(za).cpu().numpy()
    keep = o.mask.ravel() > 0
    assert rel_l2(Az[keep], r[keep]) < 1e-11


SMOOTHERS = ["jacobi", "cheby_jac", "asm", "ras", "cheby_asm", "cheby_ras"]


@pytest.mark.parametrize("smoother", SMOOTHERS)
def test_hierarchy_smoothers_match_oracle(smoother):
    N, counts = 7, (2, 2, 2)
    kw = dict(bc="dirichlet", deformation=("sine", 0.05))
    m = nk.build_box_mesh((1, 1, 1), counts, N, **kw)
    op = nk.PoissonOperator(m)
    h = nk.MultigridHierarchy(op, smoother=smoother)
    o = opmg.build_hierarchy((1, 1, 1), counts, N, smoother=smoother, **kw)
    for lg, lo in zip(h.levels[:-1], o["levels"][:-1]):
        assert abs(lg.lmax - lo.lmax) < 1e-9 * lo.lmax
    lv = o["levels"][0]
    r = lv.mask * ogs.gs_op(lv.mesh.ids, lv.wt * np.random.default_rng(7).standard_normal(
        lv.mask.size))
    z = nk.pmg_preconditioner(h, dev(r)).cpu().numpy()
    assert rel_l2(z, opmg.vcycle(o, r)) < 1e-9
    for level in (0, 1):
        lo = o["levels"][level]
        rl = lo.mask * ogs.gs_op(lo.mesh.ids, lo.wt * np.random.default_rng(level).standard_normal(
            lo.mask.size))
        e = nk.chebyshev_smooth(h, level, dev(rl)).cpu().numpy()
        assert rel_l2(e, opmg.smooth(lo, rl, o["degree"])) < 1e-10


@pytest.mark.parametrize("smoother", SMOOTHERS)
def test_flexible_pcg_iterations_match_oracle(smoother):
    N, counts = 7, (3, 3, 3)
    kw = dict(bc="dirichlet", deformation=("sine", 0.05))
    m = nk.build_box_mesh((1, 1, 1), counts, N, **kw)
    op = nk.PoissonOperator(m)
    h = nk.MultigridHierarchy(op, smoother=smoother)
    o = opmg.build_hierarchy((1, 1, 1), counts, N, smoother=smoother, **kw)
    lv = o["levels"][0]
    X = lv.mesh.xyz.reshape(3, -1)
    f = 3 * np.pi ** 2 * np.prod(np.sin(np.pi * X), axis=0)
    b = lv.mask * ogs.gs_op(lv.mesh.ids, lv.mesh.B.ravel() * f)
    ro = osol.pcg(opmg.fine_operator(o), lambda r: opmg.vcycle(o, r), b, tol=1e-8,
                  max_iter=200, flexible=True, weights=lv.wt)
    res = nk.MultigridPCG(op, h, tol=1e-8, max_iter=200, flexible=True).solve(dev(b))
    assert res.converged and ro.converged
    assert abs(res.iterations - ro.iterations) <= 1
    assert np.max(np.abs(res.x.cpu().numpy() - ro.x)) < 1e-7 * np.max(np.abs(ro.x))


def test_contract_errors():
    m = nk.build_box_mesh((1, 1, 1), (2, 2, 2), 3)
    op = nk.PoissonOperator(m)
    with pytest.raises(nk.ContractError):
        nk.SchwarzSmoother(op, "bogus")
    with pytest.raises(nk.ContractError):
        nk.MultigridHierarchy(op, smoother="bogus")
    sm = nk.SchwarzSmoother(op, "ras")
    with pytest.raises(nk.ContractError):
        sm(torch.zeros(5, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("kind", ["asm", "ras"])
@pytest.mark.parametrize("N", [3, 7, 15])
def test_fp32_local_solves_close_to_fp64(kind, N):
    """32-bit smoothing: FP32 local solves,
    FP64 fields -- within single-precision accuracy of the FP64 smoother."""
    counts = (2, 2, 2) if N < 15 else (1, 2, 1)
    m, o, op, f = pair(counts, N)
    r = dev(assembled_random(o, 5))
    z64 = nk.SchwarzSmoother(op, kind)(r).cpu().numpy()
    z32 = nk.SchwarzSmoother(op, kind, precision=32)(r).cpu().numpy()
    assert rel_l2(z32, z64) < 2e-5


@pytest.mark.parametrize("smoother", ["asm", "ras", "cheby_asm", "cheby_ras"])
def test_fp32_smoothing_iterations_within_two(smoother):
    """32-bit smoothing changes iteration counts by <= 2 and the
    converged solution meets the tolerance."""
    N, counts = 7, (3, 3, 3)
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    b = torch.randn(op.n, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(b.dtype)
    r64 = nk.MultigridPCG(op, nk.MultigridHierarchy(op, smoother=smoother), tol=1e-8,
                          max_iter=200, flexible=True).solve(b)
    x64 = r64.x.clone()
    r32 = nk.MultigridPCG(op, nk.MultigridHierarchy(op, smoother=smoother, smoother_precision=32),
                          tol=1e-8, max_iter=200, flexible=True).solve(b)
    assert r32.converged and abs(r32.iterations - r64.iterations) <= 2
    res = b - op(r32.x)
    wt = op.weights
    assert float(torch.sqrt(torch.sum(wt * res * res))) <= 1.01e-8 * float(
        torch.sqrt(torch.sum(wt * b * b)))
    assert float((r32.x - x64).abs().max()) < 1e-6 * float(x64.abs().max())


def test_fp32_contract_errors():
    m = nk.build_box_mesh((1, 1, 1), (2, 2, 2), 3)
    op = nk.PoissonOperator(m)
    with pytest.raises(nk.ContractError):
        nk.SchwarzSmoother(op, "asm", precision=16)
    with pytest.raises(nk.ContractError):
        nk.MultigridHierarchy(op, smoother="cheby_jac", smoother_precision=32)


def test_coordinate_mesh_schwarz_matches_box(tmp_path):
    """Meshes read from HEXMESH files (ids from coordinates) find the same
    face neighbours and element lengths: identical Schwarz smoothing."""
    N = 4
    mb = nk.build_box_mesh((1, 1, 1), (3, 2, 2), N, deformation=("sine", 0.05), keep_coords=True)
    path = str(tmp_path / "box.hexmesh")
    nk.write_hexmesh(path, mb.xyz.cpu().numpy(), mb.ids.cpu().numpy(),
                     {"pressure": mb.mask.cpu().numpy().ravel()})
    E, Nr, xyz, ids, masks = nk.read_hexmesh(path)
    mc = nk.mesh.mesh_from_coords(xyz, Nr, ids=ids, mask=masks["pressure"])
    r = torch.randn(mb.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(nk.PoissonOperator(mb).gs, r)
    r *= mb.mask.reshape(-1).to(r.dtype)
    for kind in ("asm", "ras"):
        zb = nk.SchwarzSmoother(nk.PoissonOperator(mb), kind)(r)
        zc = nk.SchwarzSmoother(nk.PoissonOperator(mc), kind)(r)
        assert rel_l2(zc.cpu().numpy(), zb.cpu().numpy()) < 1e-13
    # and the whole hierarchy on the coordinate mesh
    hc = nk.MultigridHierarchy(nk.PoissonOperator(mc), smoother="ras")
    z = nk.pmg_preconditioner(hc, r)
    assert torch.isfinite(z).all() and float(z.abs().max()) > 0


@pytest.mark.parametrize("smoother", ["asm", "ras", "cheby_ras"])
@pytest.mark.parametrize("bc,lam1", [("periodic", 5.0), ("neumann", 3.0),
                                     ({"x-": "dirichlet", "y+": "dirichlet"}, 0.0)])
def test_hierarchy_schwarz_boundary_kinds_match_oracle(smoother, bc, lam1):
    """Schwarz-smoothed V-cycles on periodic / Neumann (Helmholtz) / mixed
    boundaries -- every side kind of the FDM surrogate ('nbr', 'neu', 'dir')
    -- against the oracle hierarchy."""
    N, counts = 5, (3, 2, 2)
    kw = dict(bc=bc, deformation=("sine", 0.05) if bc != "periodic" else None)
    m = nk.build_box_mesh((1, 1, 1), counts, N, **kw)
    op = nk.PoissonOperator(m, lam0=1.0, lam1=lam1)
    h = nk.MultigridHierarchy(op, smoother=smoother)
    o = opmg.build_hierarchy((1, 1, 1), counts, N, smoother=smoother, lam0=1.0, lam1=lam1, **kw)
    for lg, lo in zip(h.levels[:-1], o["levels"][:-1]):
        assert abs(lg.lmax - lo.lmax) < 1e-9 * lo.lmax
    lv = o["levels"][0]
    r = lv.mask * ogs.gs_op(lv.mesh.ids, lv.wt * np.random.default_rng(3).standard_normal(
        lv.mask.size))
    z = nk.pmg_preconditioner(h, dev(r)).cpu().numpy()
    assert rel_l2(z, opmg.vcycle(o, r)) < 1e-9


@pytest.mark.parametrize("N", [2, 3, 4, 6, 9, 10, 15])
def test_ras_hierarchy_all_orders_match_oracle(N):
    """p-multigrid with RAS smoothing at low and high orders (every
    specialised transfer pair N+1 <-> N/2+1 <-> 2): λmax and the V-cycle vs
    the oracle."""
    counts = (2, 2, 1) if N < 10 else (1, 2, 1)
    kw = dict(bc="dirichlet", deformation=("sine", 0.05))
    m = nk.build_box_mesh((1, 1, 1), counts, N, **kw)
    op = nk.PoissonOperator(m)
    h = nk.MultigridHierarchy(op, smoother="ras")
    o = opmg.build_hierarchy((1, 1, 1), counts, N, smoother="ras", **kw)
    assert h.orders == opmg.orders_for(N)
    for lg, lo in zip(h.levels[:-1], o["levels"][:-1]):
        assert abs(lg.lmax - lo.lmax) < 1e-9 * lo.lmax
    lv = o["levels"][0]
    r = lv.mask * ogs.gs_op(lv.mesh.ids, lv.wt * np.random.default_rng(N).standard_normal(
        lv.mask.size))
    z = nk.pmg_preconditioner(h, dev(r)).cpu().numpy()
    assert rel_l2(z, opmg.vcycle(o, r)) < 1e-9
