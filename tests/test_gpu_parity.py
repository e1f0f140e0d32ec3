"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): gs index map bit-exact; Ax within 1e-12
relative L2 (FP64); PCG iterations within +-1 at the same tolerance.
"""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om
from oracle import operators as oop
from oracle import solvers as osol

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import _lib  # noqa: E402

BK5_TOL = 1e-12   # relative L2, FP64 (north_star)


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def both_meshes(counts, N, bc="dirichlet", deformation=("sine", 0.05), extent=(1.0, 1.0, 1.0)):
    return (nk.build_box_mesh(extent, counts, N, bc=bc, deformation=deformation,
                              keep_coords=True, keep_jacobian=True),
            om.build_box_mesh(extent, counts, N, bc=bc, deformation=deformation))


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


# ---------------------------------------------------------------- geometry
@pytest.mark.parametrize("N", [1, 3, 7, 10])
def test_geometry_matches_oracle(N):
    m, o = both_meshes((3, 2, 2), N)
    xyz = m.xyz.cpu().numpy()
    assert np.max(np.abs(xyz - o.xyz)) < 1e-14
    G = m.G.cpu().numpy()
    assert rel_l2(G, o.G) < 1e-13
    assert rel_l2(m.B.cpu().numpy(), o.B) < 1e-13
    assert rel_l2(m.J.cpu().numpy(), o.J) < 1e-13
    assert np.array_equal(m.ids.cpu().numpy(), o.ids)                    # bit-exact ids
    assert np.array_equal(m.mask.cpu().numpy().astype(float), o.mask)


@pytest.mark.parametrize("bc", ["periodic", "neumann", ("dirichlet", "neumann", "periodic",
                                                          "periodic", "neumann", "dirichlet")])
def test_ids_and_mask_bc(bc):
    m, o = both_meshes((4, 3, 2), 3, bc=bc, deformation=None)
    assert np.array_equal(m.ids.cpu().numpy(), o.ids)
    assert np.array_equal(m.mask.cpu().numpy().astype(float), o.mask)


def test_geometric_factors_single_element():
    b = nk.SpectralBasis.get(2)
    o = om.build_box_mesh((2, 2, 2), (1, 1, 1), 2, bc="neumann", origin=(-1, -1, -1))
    J, rx, G, B = nk.geometric_factors(o.xyz[:, 0], b)
    assert np.allclose(J, 1.0) and np.allclose(G[[1, 2, 4]], 0.0)
    for q in range(3):
        for p in range(3):
            assert np.allclose(rx[q, p], 1.0 if p == q else 0.0)


def test_inverted_element_raises():
    with pytest.raises(nk.mesh.InvertedElementError):
        nk.build_box_mesh((1, 1, 1), (2, 2, 2), 3,
                          deformation=lambda x, y, z: (-x, y, z))


# ---------------------------------------------------------------- BK5
@pytest.mark.parametrize("N", list(range(1, 16)))
def test_bk5_all_orders(N):
    counts = (3, 2, 2) if N <= 9 else (2, 2, 1)
    m, o = both_meshes(counts, N)
    rng = np.random.default_rng(1000 + N)
    u = rng.standard_normal((m.E, N + 1, N + 1, N + 1))
    w = nk.apply_stiffness_local(dev(u), m).cpu().numpy()
    w_ref = oop.bk5(o.basis.diff, o.G, u)
    assert rel_l2(w, w_ref) < BK5_TOL


@pytest.mark.parametrize("N", [3, 7, 9])
def test_bk5_helmholtz_and_batched(N):
    m, o = both_meshes((2, 2, 2), N)
    rng = np.random.default_rng(5 + N)
    u = rng.standard_normal((3, m.E, N + 1, N + 1, N + 1))
    lam0, lam1 = 1e-3, 11 / 6 / 1e-3
    w = nk.apply_helmholtz_local(dev(u), m, lam0, lam1, ncomp=3).cpu().numpy()
    for c in range(3):
        ref = oop.bk5(o.basis.diff, o.G, u[c], lam0=lam0, B=o.B, lam1=lam1)
        assert rel_l2(w[c], ref) < BK5_TOL
    w1 = nk.apply_helmholtz_local(dev(u[1]), m, lam0, lam1).cpu().numpy()
    assert rel_l2(w1, oop.bk5(o.basis.diff, o.G, u[1], lam0=lam0, B=o.B, lam1=lam1)) < BK5_TOL


@pytest.mark.parametrize("N", list(range(1, 16)))
def test_bk5_helmholtz3_auto_and_seq3(N):
    """3-component batches at every order: the auto table (seq3 / pencil3 /
    three scalar launches, bk5.cu) vs the oracle, and the seq3 kernel
    (bk5_pencil NC = 3) bitwise equal to three scalar pencil launches."""
    from paper_2104_05829_b200 import kernels as K
    from paper_2104_05829_b200._lib import lib
    counts = (3, 2, 2) if N <= 9 else (2, 2, 1)
    m, o = both_meshes(counts, N)
    rng = np.random.default_rng(50 + N)
    u = rng.standard_normal((3, m.E, N + 1, N + 1, N + 1))
    lam0, lam1 = 0.7, 2.5
    w = nk.apply_helmholtz_local(dev(u), m, lam0, lam1, ncomp=3).cpu().numpy()
    for c in range(3):
        ref = oop.bk5(o.basis.diff, o.G, u[c], lam0=lam0, B=o.B, lam1=lam1)
        assert rel_l2(w[c], ref) < BK5_TOL
    try:
        lib().nk_bk5_set_variant(K.BK5_VARIANTS["seq3"])
        ws = nk.apply_helmholtz_local(dev(u), m, lam0, lam1, ncomp=3).cpu().numpy()
        lib().nk_bk5_set_variant(K.BK5_VARIANTS["pencil"])
        w1 = [nk.apply_helmholtz_local(dev(u[c]), m, lam0, lam1).cpu().numpy() for c in range(3)]
    finally:
        lib().nk_bk5_set_variant(0)
    for c in range(3):
        assert rel_l2(ws[c], oop.bk5(o.basis.diff, o.G, u[c], lam0=lam0, B=o.B, lam1=lam1)) < BK5_TOL
        if N > 1:   # N = 1 scalar calls run bk5_n1, not the pencil kernel
            assert np.array_equal(ws[c], w1[c])


def test_bk5_element_subset():
    N = 7
    m, o = both_meshes((3, 3, 2), N)
    rng = np.random.default_rng(7)
    u = rng.standard_normal((m.E, 8, 8, 8))
    sub = np.array([0, 5, 17, 3], dtype=np.int32)
    w = torch.full((m.E, 8, 8, 8), 7.0, dtype=torch.float64, device="cuda")
    nk.apply_stiffness_local(dev(u), m, out=w, elements=dev(sub))
    w = w.cpu().numpy()
    ref = oop.bk5(o.basis.diff, o.G, u)
    assert rel_l2(w[sub], ref[sub]) < BK5_TOL
    rest = np.setdiff1d(np.arange(m.E), sub)
    assert np.all(w[rest] == 7.0)


def test_bk5_config2_size_n7():
    """Full configs[1] size at N=7 (E = 20^3, 4.1M local points)."""
    N = 7
    m, o = both_meshes((20, 20, 20), N)
    rng = np.random.default_rng(1007)
    u = rng.standard_normal((m.E, 8, 8, 8))
    w = nk.apply_stiffness_local(dev(u), m).cpu().numpy()
    ref = oop.bk5(o.basis.diff, o.G, u)
    assert rel_l2(w, ref) < BK5_TOL
    # Neumann-nullspace property at full size: Q^T A_L Q 1 = 0
    mn = nk.build_box_mesh((1, 1, 1), (20, 20, 20), N, bc="neumann", deformation=("sine", 0.05))
    one = torch.ones((mn.E, 8, 8, 8), dtype=torch.float64, device="cuda")
    h = nk.gs_setup(mn.ids, nq=8)
    a1 = nk.gs_op(h, nk.apply_stiffness_local(one, mn))
    scale = nk.gs_op(h, nk.apply_stiffness_local(dev(u), mn)).abs().max().item()
    assert a1.abs().max().item() < 1e-11 * scale


def test_bk5_contract_errors():
    m, _ = both_meshes((1, 1, 1), 3)
    with pytest.raises(nk.ContractError):
        nk.apply_stiffness_local(torch.zeros(5, dtype=torch.float64, device="cuda"), m)
    with pytest.raises(nk.ContractError):
        nk.apply_stiffness_local(torch.zeros(64, dtype=torch.float64, device="cuda"), m,
                                 basis=nk.SpectralBasis.get(4))


def test_local_diag_matches_oracle():
    for N in (2, 7, 11):
        m, o = both_meshes((2, 2, 1), N)
        d = nk.extract_diagonal(m, assemble=False).cpu().numpy()
        assert rel_l2(d, oop.local_diagonal(o.basis.diff, o.G)) < 1e-13
        d = nk.extract_diagonal(m, spec=("helmholtz", 0.5, 3.0)).cpu().numpy()
        ref = ogs.gs_op(o.ids, oop.local_diagonal(o.basis.diff, o.G, 0.5, o.B, 3.0).ravel())
        assert rel_l2(d, ref) < 1e-13


# ---------------------------------------------------------------- gather-scatter
@pytest.mark.parametrize("bc,N,counts", [("dirichlet", 7, (4, 4, 4)), ("periodic", 3, (3, 4, 5)),
                                         ("periodic", 1, (2, 2, 2)), ("neumann", 7, (20, 20, 20))])
def test_gs_map_and_values_bit_exact(bc, N, counts):
    m, o = both_meshes(counts, N, bc=bc, deformation=None)
    h = nk.gs_setup(m.ids, nq=N + 1)
    perm, seg = h.plan_host()
    operm, oseg = ogs.local_plan(o.ids)
    assert np.array_equal(perm, operm) and np.array_equal(seg, oseg)
    rng = np.random.default_rng(N)
    w = rng.standard_normal(o.ids.size)
    for op in ("+", "*", "min", "max"):
        got = nk.gs_op(h, dev(w.copy()), op).cpu().numpy()
        assert np.array_equal(got, ogs.gs_op(o.ids, w, op)), op


def test_gs_random_topologies_vs_dense():
    rng = np.random.default_rng(11)
    for t in range(30):
        n = int(rng.integers(1, 400))
        ids = rng.integers(0, max(2, n // 3), size=n)
        w = rng.standard_normal(n)
        h = nk.gs_setup(ids)
        got = nk.gs_op(h, dev(w.copy())).cpu().numpy()
        assert np.array_equal(got, ogs.gs_op(ids, w))
        Q = ogs.dense_Q(ids)
        assert np.allclose(got, Q @ (Q.T @ w), atol=1e-12)


def test_gs_numpy_roundtrip_and_errors():
    h = nk.gs_setup(np.array([5, 5, 0]))
    assert np.array_equal(nk.gs_op(h, np.array([3.5, 3.5, 1.0])), [7.0, 7.0, 1.0])
    with pytest.raises(nk.ContractError):
        nk.gs_op(h, np.zeros(4))
    h0 = nk.gs_setup(np.zeros(6, dtype=np.int64))
    x = np.arange(6.0)
    assert np.array_equal(nk.gs_op(h0, x.copy()), x)


# ---------------------------------------------------------------- PCG
def _oracle_problem(o):
    X = o.xyz.reshape(3, -1)
    f = 3 * np.pi ** 2 * np.prod(np.sin(np.pi * X), axis=0)
    mask = o.mask.ravel()
    b = mask * ogs.gs_op(o.ids, o.B.ravel() * f)
    D, G = o.basis.diff, o.G
    sh = (o.G.shape[0],) + o.G.shape[2:]

    def A(v):
        return mask * ogs.gs_op(o.ids, oop.bk5(D, G, v.reshape(sh)).ravel())

    inv = mask / ogs.gs_op(o.ids, oop.local_diagonal(D, G).ravel())
    return b, A, inv, 1.0 / ogs.multiplicity(o.ids)


@pytest.mark.parametrize("deform", [None, ("sine", 0.05)])
def test_pcg_config1_iterations(deform):
    """configs[0]: BP5 on the 4x4x4 box, N=7, Jacobi, tol 1e-8."""
    m, o = both_meshes((4, 4, 4), 7, deformation=deform)
    b, A, inv, wt = _oracle_problem(o)
    ref = osol.pcg(A, lambda r: inv * r, b, tol=1e-8, max_iter=1000, weights=wt)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    res = nk.pcg(op, jac, dev(b), tol=1e-8, max_iter=1000)
    assert res.converged and ref.converged
    assert abs(res.iterations - ref.iterations) <= 1
    assert np.max(np.abs(res.x.cpu().numpy() - ref.x)) < 1e-7 * np.max(np.abs(ref.x))
    assert len(res.residual_history) == res.iterations + 1
    # random rhs variant
    rng = np.random.default_rng(2104_05829)
    br = o.mask.ravel() * ogs.gs_op(o.ids, rng.standard_normal(o.ids.size))
    ref = osol.pcg(A, lambda r: inv * r, br, tol=1e-8, max_iter=1000, weights=wt)
    res = nk.pcg(op, jac, dev(br), tol=1e-8, max_iter=1000)
    assert abs(res.iterations - ref.iterations) <= 1


def test_pcg_generic_and_flexible():
    m, o = both_meshes((3, 3, 3), 5)
    b, A, inv, wt = _oracle_problem(o)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    ref = osol.pcg(A, lambda r: inv * r, b, tol=1e-9, max_iter=500, weights=wt)
    gen = nk.pcg(lambda v: op(v), lambda r: jac(r), dev(b), tol=1e-9, max_iter=500,
                 weights=op.weights)
    assert abs(gen.iterations - ref.iterations) <= 1
    assert np.max(np.abs(gen.x.cpu().numpy() - ref.x)) < 1e-7
    flex = nk.pcg(op, jac, dev(b), tol=1e-9, max_iter=500, flexible=True)
    assert abs(flex.iterations - ref.iterations) <= 1
    # non-convergence flag with the last iterate
    short = nk.pcg(op, jac, dev(b), tol=1e-14, max_iter=5)
    assert not short.converged and short.iterations == 5


def test_pcg_spec_examples():
    d = torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64, device="cuda")
    r = nk.pcg(lambda v: d * v, lambda v: v / d, torch.ones(3, dtype=torch.float64, device="cuda"),
               tol=1e-12)
    assert r.iterations == 1 and np.allclose(r.x.cpu().numpy(), 1 / d.cpu().numpy())
    z = nk.pcg(lambda v: v, lambda v: v, torch.zeros(4, dtype=torch.float64, device="cuda"))
    assert z.iterations == 0 and z.converged
    with pytest.raises(nk.BreakdownError):
        nk.pcg(lambda v: -v, lambda v: v, torch.ones(3, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("counts,N", [((4, 4, 4), 7), ((10, 10, 10), 7), ((3, 3, 3), 5),
                                      ((3, 2, 3), 3)])
def test_launch_knobs_bit_identical(counts, N):
    """PDL (programmatic dependent launch with static-operand prologues), the
    update's L2 prefetch and the L2 eviction hints change scheduling / cache
    policy only: solves with every knob off, at the defaults and with every
    option on are bit-identical, graph-captured included."""
    from paper_2104_05829_b200._lib import lib
    L = lib()
    m, o = both_meshes(counts, N)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    rng = np.random.default_rng(90 + N)
    b = torch.as_tensor(o.mask.ravel() * ogs.gs_op(o.ids, rng.standard_normal(m.n_local)),
                        device="cuda")
    ra = nk.FusedPCG(op, jac, tol=1e-9, max_iter=3000).solve(b)
    old = (L.nk_set_knob(0, 0), L.nk_set_knob(1, 0), L.nk_set_knob(2, 0))
    try:
        rb = nk.FusedPCG(op, jac, tol=1e-9, max_iter=3000).solve(b)
        L.nk_set_knob(0, 31)      # every PDL family, late trigger, no prologue
        L.nk_set_knob(2, 7)       # every L2 hint
        rc = nk.FusedPCG(op, jac, tol=1e-9, max_iter=3000).solve(b)
    finally:
        for k, v in enumerate(old):
            L.nk_set_knob(k, v)
    for r in (rb, rc):
        assert r.iterations == ra.iterations and r.residual_history == ra.residual_history
        assert torch.equal(r.x, ra.x)


@pytest.mark.parametrize("counts,N,lam1,split", [((5, 4, 4), 1, 0.0, None),
                                                 ((3, 3, 3), 2, 0.0, None),  # odd n
                                                 ((3, 2, 3), 3, 0.5, None),
                                                 ((4, 4, 4), 7, 0.0, False),
                                                 ((4, 4, 4), 7, 0.0, True),
                                                 ((10, 10, 10), 7, 0.0, False),  # ring reuse
                                                 ((2, 3, 2), 8, 0.0, None),
                                                 ((2, 2, 2), 12, 0.3, None)])
def test_fused_pcg_gathered_segments(counts, N, lam1, split):
    """gather_segments (nk_cg_update_gs_seg: every member of an edge /
    vertex segment folds the segment in canonical order inside the update,
    no gs pass) against the gs sub-plan + nk_cg_update_gs: bit-identical
    solves (iterations, residual history, x), one launch fewer."""
    m, o = both_meshes(counts, N)
    op = nk.PoissonOperator(m, lam1=lam1)
    jac = nk.JacobiPreconditioner(op)
    rng = np.random.default_rng(70 + N)
    b = torch.as_tensor(o.mask.ravel() * ogs.gs_op(o.ids, rng.standard_normal(m.n_local)),
                        device="cuda")
    sa = nk.FusedPCG(op, jac, tol=1e-9, max_iter=3000, split_step=split, gather_segments=True)
    sb = nk.FusedPCG(op, jac, tol=1e-9, max_iter=3000, split_step=split)
    assert sa.gcodes is not None and sb.gcodes is None
    assert sa.launches_per_iter == sb.launches_per_iter - 1
    ra, rb = sa.solve(b), sb.solve(b)
    assert ra.converged and ra.iterations == rb.iterations
    assert ra.residual_history == rb.residual_history
    assert torch.equal(ra.x, rb.x)
    if m.E <= 64 and lam1 == 0.0:
        _, A, inv, wt = _oracle_problem(o)
        ref = osol.pcg(A, lambda r: inv * r, b.cpu().numpy(), tol=1e-9, max_iter=3000,
                       weights=wt)
        assert abs(ra.iterations - ref.iterations) <= 1
        assert np.max(np.abs(ra.x.cpu().numpy() - ref.x)) < 1e-7 * np.max(np.abs(ref.x))


@pytest.mark.parametrize("counts,N,lam1", [((5, 4, 4), 1, 0.0), ((3, 3, 2), 2, 0.0),
                                           ((3, 3, 3), 2, 0.0),   # n = 729: odd tail
                                           ((3, 2, 3), 3, 0.5),
                                           ((4, 4, 4), 7, 0.0), ((2, 3, 2), 8, 0.0),
                                           ((2, 2, 2), 12, 0.3)])
def test_fused_pcg_split_step(counts, N, lam1):
    """split_step (nk_cg_xpstep + nk_bk5 with the fused p.Ap) against the
    one-kernel fused step: with the pencil kernel forced on both paths the
    solves are bit-identical (same iterations, residual history, x); in auto
    mode the split is the default at N != 7 and solves the system."""
    from paper_2104_05829_b200 import kernels as K
    from paper_2104_05829_b200._lib import lib
    m, o = both_meshes(counts, N)
    op = nk.PoissonOperator(m, lam1=lam1)
    jac = nk.JacobiPreconditioner(op)
    rng = np.random.default_rng(40 + N)
    b = torch.as_tensor(o.mask.ravel() * ogs.gs_op(o.ids, rng.standard_normal(m.n_local)),
                        device="cuda")
    try:
        lib().nk_bk5_set_variant(K.BK5_VARIANTS["pencil"])
        sa = nk.FusedPCG(op, jac, tol=1e-9, max_iter=3000, split_step=True)
        sb = nk.FusedPCG(op, jac, tol=1e-9, max_iter=3000, split_step=False)
        assert sa.split and sa.launches_per_iter == 4 and not sb.split
        ra, rb = sa.solve(b), sb.solve(b)
    finally:
        lib().nk_bk5_set_variant(0)
    assert ra.converged and abs(ra.iterations - rb.iterations) <= (1 if N == 1 else 0)
    if N > 1:   # N = 1 runs the point-per-lane kernels (bk5_n1 vs bk5_n1_pcg)
        assert ra.residual_history == rb.residual_history
        assert torch.equal(ra.x, rb.x)
    sc = nk.FusedPCG(op, jac, tol=1e-9, max_iter=3000)
    assert sc.split == (N not in nk.solvers.SPLIT_STEP_OFF and
                        m.n_local >= nk.solvers.split_min_points(N))
    rc = sc.solve(b)
    assert rc.converged and abs(rc.iterations - rb.iterations) <= 1
    Ax = torch.empty_like(b)
    op(rc.x.reshape(-1), out=Ax)
    assert float(torch.linalg.norm(Ax - b)) <= 2e-9 * float(torch.linalg.norm(b))
    keys = ({"cg_xpstep", "bk5"} if sc.split else {"bk5_pcg"}) | {"cg_update_gs"}
    if sc.gcodes is None:
        keys |= {"gs_nonpair"}
    assert set(sc.profile_iteration(reps=2)) == keys
    assert len(keys) == sc.launches_per_iter


def test_fused_pcg_deterministic_and_graph_equivalent():
    m, o = both_meshes((4, 4, 4), 7)
    b, _, _, _ = _oracle_problem(o)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    s1 = nk.FusedPCG(op, jac, tol=1e-8, chunk=7)
    r1 = s1.solve(dev(b))
    x1 = r1.x.cpu().numpy().copy()
    r2 = s1.solve(dev(b))
    assert r1.iterations == r2.iterations and np.array_equal(x1, r2.x.cpu().numpy())
    s3 = nk.FusedPCG(op, jac, tol=1e-8, chunk=3, use_graph=False)
    r3 = s3.solve(dev(b))
    assert r3.iterations == r1.iterations and np.array_equal(x1, r3.x.cpu().numpy())


@pytest.mark.parametrize("counts,N,bc,lam1", [((4, 4, 4), 7, "dirichlet", 0.0),
                                              ((3, 4, 2), 3, "periodic", 1.0),
                                              ((6, 5, 4), 1, "dirichlet", 0.0),
                                              ((3, 3, 3), 2, "neumann", 0.5),
                                              ((2, 2, 3), 12, "dirichlet", 0.0)])
def test_fused_gs_update_bit_identical(counts, N, bc, lam1):
    """nk_cg_update_gs (face pairs folded into the CG update, gs pass over
    edge/vertex segments only) against the full-gs schedule (bk5_pcg, gs,
    cg_update): same iterations, residual history and solution bit for bit;
    and the answer solves the system."""
    m, o = both_meshes(counts, N, bc=bc)
    op = nk.PoissonOperator(m, lam1=lam1)
    jac = nk.JacobiPreconditioner(op)
    rng = np.random.default_rng(N)
    b = torch.as_tensor(o.mask.ravel() * ogs.gs_op(o.ids, rng.standard_normal(m.n_local)),
                        device="cuda")
    s2 = nk.FusedPCG(op, jac, tol=1e-9, max_iter=2000, split_step=False)
    assert s2.codes is not None and s2.launches_per_iter == (2 if s2.gs_tail else 3)
    s3 = nk.FusedPCG(op, jac, tol=1e-9, max_iter=2000, fuse_gs=False)
    assert s3.codes is None
    r2, r3 = s2.solve(b), s3.solve(b)
    assert r2.converged and r2.iterations == r3.iterations
    assert r2.residual_history == r3.residual_history
    assert torch.equal(r2.x, r3.x)
    Ax = torch.empty_like(b)
    op(r2.x.reshape(-1), out=Ax)
    assert float(torch.linalg.norm(Ax - b)) <= 2e-9 * float(torch.linalg.norm(b))
    prof = s2.profile_iteration(reps=2)
    assert set(prof) == ({"bk5_pcg", "cg_update_gs"} if s2.gs_tail else
                         {"bk5_pcg", "gs_nonpair", "cg_update_gs"})


def test_native_library_loaded():
    import os
    assert os.path.exists(_lib.LIB_PATH)
    L = _lib.lib()
    sm = np.zeros(1, np.int32)
    l2 = np.zeros(1, np.int64)
    mj = np.zeros(1, np.int32)
    mi = np.zeros(1, np.int32)
    _lib.check(L.nk_device_info(sm.ctypes.data, l2.ctypes.data, mj.ctypes.data, mi.ctypes.data))
    assert mj[0] >= 10


# ---------------------------------------------------------------- kernel variants
@pytest.fixture
def variant_guard():
    L = _lib.lib()
    old = L.nk_bk5_set_variant(0)
    yield L
    L.nk_bk5_set_variant(old)
    L.nk_bk5_tune(0, 1)


@pytest.mark.parametrize("variant", [1, 3, 4, 5])
@pytest.mark.parametrize("N", [1, 2, 3, 5, 7, 12])
def test_bk5_variants_match_oracle(variant_guard, variant, N):
    """k-slab (1), pencil (3), pencil-TMA (4, even N+1; others fall back),
    pencil2 (5; N = 1 has its own point-per-lane kernel) all within the 1e-12 bar, incl. element subsets, mask and the fused p.Ap."""
    L = variant_guard
    L.nk_bk5_set_variant(variant)
    m, o = both_meshes((5, 4, 3), N)
    rng = np.random.default_rng(77 + N)
    u = rng.standard_normal((m.E, N + 1, N + 1, N + 1))
    w = nk.apply_stiffness_local(dev(u), m).cpu().numpy()
    ref = oop.bk5(o.basis.diff, o.G, u)
    assert rel_l2(w, ref) < BK5_TOL
    sub = np.array([7, 0, 59, 31, 2], dtype=np.int32)
    w2 = torch.zeros((m.E, N + 1, N + 1, N + 1), dtype=torch.float64, device="cuda")
    nk.apply_stiffness_local(dev(u), m, out=w2, elements=dev(sub))
    assert rel_l2(w2.cpu().numpy()[sub], ref[sub]) < BK5_TOL
    # fused p.Ap via the PoissonOperator path (masked, assembled)
    op = nk.PoissonOperator(m)
    st = torch.zeros(_lib.CG_STATE_BYTES, dtype=torch.uint8, device="cuda")
    part = torch.zeros(op.partials_len(), dtype=torch.float64, device="cuda")
    p = dev(o.mask * ogs.gs_op(o.ids, u.ravel()).reshape(u.shape))
    Ap = torch.empty_like(p)
    op.apply(p, Ap, st=st, partials=part)
    pAp = nk.solvers.read_state(st).pAp
    pn = p.cpu().numpy().ravel()
    ref_Ap = o.mask.ravel() * ogs.gs_op(o.ids, oop.bk5(o.basis.diff, o.G, pn.reshape(u.shape)).ravel())
    assert rel_l2(Ap.cpu().numpy().ravel(), ref_Ap) < BK5_TOL
    ref_pAp = float(np.sum(pn * ref_Ap / ogs.multiplicity(o.ids)))
    assert abs(pAp - ref_pAp) < 1e-11 * abs(ref_pAp)


def test_host_streamed_apply_matches_device_path():
    """numpy / pinned-host input goes through the chunked host pipeline (direct
    mode at N = 7: the stage kernel writes w into host memory; else H2D-BK5-D2H
    copies); results must equal the device path bit for bit."""
    N = 7
    m, o = both_meshes((5, 3, 2), N)
    rng = np.random.default_rng(3)
    u = rng.standard_normal((m.E, 8, 8, 8))
    wd = nk.apply_stiffness_local(dev(u), m).cpu().numpy()
    wn = nk.apply_stiffness_local(u, m)                         # numpy in -> numpy out
    assert isinstance(wn, np.ndarray) and np.array_equal(wn, wd)
    uh = torch.as_tensor(u).pin_memory()
    wh = torch.empty_like(uh).pin_memory()
    from paper_2104_05829_b200 import kernels as K
    saved, saved_stream = K._HostStream.DIRECT_ORDERS, K._HostStream.STREAM
    try:
        # N = 7: stream mode (one chunk-gated stage kernel), direct mode (one
        # stage kernel per chunk; both bulk-store w into the pinned host w),
        # then the H2D / BK5 / D2H copy pipeline; every case twice (the
        # second call replays the cached graph: the gate must be re-armed)
        for direct, stream in ((saved, True), (saved, False), ((), False)):
            K._HostStream.DIRECT_ORDERS = direct
            K._HostStream.STREAM = stream
            m._host_stream = None
            for chunks in (None, 1, 7, 30):
                for _ in range(2):
                    wh.zero_()
                    nk.apply_stiffness_local(uh, m, out=wh, nchunks=chunks)
                    assert np.array_equal(wh.numpy(), wd), (direct, stream, chunks)
    finally:
        K._HostStream.DIRECT_ORDERS, K._HostStream.STREAM = saved, saved_stream
        m._host_stream = None
    assert rel_l2(wd, oop.bk5(o.basis.diff, o.G, u)) < BK5_TOL


def test_helmholtz_vector_solve_config5_scaled():
    """configs[4] scaled to one GPU: 3-component Helmholtz, N=9,
    lam0 = 1/Re (Re=1000), lam1 = beta0/dt (11/6 / 1e-3), rhs default_rng(5+c),
    tol 1e-6; per-component iterations within +-1 of the oracle."""
    N = 9
    m, o = both_meshes((3, 3, 3), N)
    lam0, lam1 = 1e-3, (11.0 / 6.0) / 1e-3
    solver = nk.HelmholtzVectorSolver(m, lam0, lam1, tol=1e-6)
    mask = o.mask.ravel()
    sh = (o.G.shape[0],) + o.G.shape[2:]
    bs = np.stack([mask * ogs.gs_op(o.ids, np.random.default_rng(5 + c).standard_normal(o.ids.size))
                   for c in range(3)])
    x3, res = solver.solve(dev(bs.reshape((3,) + sh)))
    D, G, B = o.basis.diff, o.G, o.B
    A = lambda v: mask * ogs.gs_op(o.ids, oop.bk5(D, G, v.reshape(sh), lam0, B, lam1).ravel())
    inv = mask / ogs.gs_op(o.ids, oop.local_diagonal(D, G, lam0, B, lam1).ravel())
    wt = 1.0 / ogs.multiplicity(o.ids)
    x3h = x3.cpu().numpy().reshape(3, -1)
    for c in range(3):
        ref = osol.pcg(A, lambda r: inv * r, bs[c], tol=1e-6, max_iter=1000, weights=wt)
        assert res[c].converged and abs(res[c].iterations - ref.iterations) <= 1
        assert np.max(np.abs(x3h[c] - ref.x)) < 1e-9 * max(1.0, np.max(np.abs(ref.x)))
    # batched operator == per-component operator
    u3 = dev(np.stack([o.mask * np.random.default_rng(c).standard_normal(sh) for c in range(3)]))
    w3 = solver.apply(u3).cpu().numpy().reshape(3, -1)
    for c in range(3):
        ref = A(u3[c].cpu().numpy().ravel())
        assert rel_l2(w3[c], ref) < BK5_TOL


def test_hexmesh_loaded_mesh_on_device(tmp_path):
    """HEXMESH v1 -> mesh_from_coords (device geometry, coordinate-snapped ids)
    -> BK5 + gs; equals the generated mesh's results."""
    N = 4
    m, o = both_meshes((3, 2, 2), N, deformation=("sine", 0.05))
    p = tmp_path / "box.hex"
    nk.write_hexmesh(p, o.xyz, o.ids, {"pressure": o.mask.astype(int)})
    E, NN, xyz, ids, masks = nk.read_hexmesh(p)
    mf = nk.mesh.mesh_from_coords(xyz, NN, ids=None, mask=masks["pressure"])
    fid = mf.ids.cpu().numpy()
    # same coincidence classes (numbering follows deformed-coordinate order)
    pairs = np.unique(np.stack([fid, o.ids]), axis=1)
    assert pairs.shape[1] == len(np.unique(fid)) == len(np.unique(o.ids))
    assert rel_l2(mf.G.cpu().numpy(), o.G) < 1e-13
    rng = np.random.default_rng(9)
    u = rng.standard_normal((E, N + 1, N + 1, N + 1))
    w = nk.apply_stiffness_local(dev(u), mf).cpu().numpy()
    assert rel_l2(w, oop.bk5(o.basis.diff, o.G, u)) < BK5_TOL


def test_gs_op_overlapped_single_rank():
    """overlapped == local_work on everything then gs_op."""
    N = 5
    m, o = both_meshes((3, 3, 2), N)
    h = nk.gs_setup(m.ids, nq=N + 1)
    rng = np.random.default_rng(4)
    u = dev(rng.standard_normal((m.E, N + 1, N + 1, N + 1)))
    field = torch.zeros_like(u)

    def local_work(elems):
        nk.apply_stiffness_local(u, m, out=field, elements=elems)

    nk.gs_op_overlapped(h, local_work, field)
    ref = ogs.gs_op(o.ids, oop.bk5(o.basis.diff, o.G, u.cpu().numpy()).ravel())
    assert rel_l2(field.cpu().numpy().ravel(), ref) < BK5_TOL


def test_fused_pcg_u8_multiplicity_weights():
    m, o = both_meshes((4, 4, 4), 7)
    b, _, _, _ = _oracle_problem(o)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    s1 = nk.FusedPCG(op, jac, tol=1e-8, fuse_gs=False)
    r1 = s1.solve(dev(b))
    x1 = r1.x.cpu().numpy().copy()
    s2 = nk.FusedPCG(op, jac, tol=1e-8, fuse_gs=False)
    s2.wt, s2.mult = None, op.multiplicity_u8
    r2 = s2.solve(dev(b))
    assert r1.iterations == r2.iterations
    assert np.max(np.abs(x1 - r2.x.cpu().numpy())) < 1e-12 * np.max(np.abs(x1))


# ---------------------------------------------------------------- edge cases
def test_edge_empty_and_ragged():
    N = 3
    m, o = both_meshes((2, 2, 1), N)
    u = dev(np.random.default_rng(0).standard_normal((m.E, 4, 4, 4)))
    w = torch.full_like(u, 3.0)
    nk.apply_stiffness_local(u, m, out=w, elements=torch.zeros(0, dtype=torch.int32,
                                                                 device="cuda"))
    assert torch.all(w == 3.0)                       # empty element list: no-op
    h = nk.gs_setup(np.zeros(0, dtype=np.int64))
    assert h.nseg == 0
    nk.gs_op(h, torch.zeros(0, dtype=torch.float64, device="cuda"))
    with pytest.raises(nk.UnsupportedOrderError):
        from paper_2104_05829_b200._lib import check, lib, ptr
        check(lib().nk_bk5(16, 1, ptr(np.zeros(289)), 1, 1, 1, 1.0, None, 0.0, 1, 1, None, None,
                           0, None, None, 0, 0, None), "bk5")
    with pytest.raises(nk.ContractError):
        nk.apply_stiffness_local(u.float(), m)


def test_edge_gs_large_multiplicities_and_many_classes():
    """multiplicity up to 40 (> 32: CSR remainder path) and > 16 distinct
    multiplicities (class table overflow) stay bit-exact."""
    rng = np.random.default_rng(21)
    ids = []
    for g, mult in enumerate(list(range(1, 41)) + [2, 3, 5, 7] * 50, start=1):
        ids += [g] * mult
    ids = np.array(ids, dtype=np.int64)
    rng.shuffle(ids)
    w = rng.standard_normal(ids.size)
    h = nk.gs_setup(ids)
    assert h.plan.rest is not None
    for op in ("+", "*", "min", "max"):
        got = nk.gs_op(h, dev(w.copy()), op).cpu().numpy()
        assert np.array_equal(got, ogs.gs_op(ids, w, op)), op


def test_edge_fused_pcg_zero_rhs_and_all_dirichlet():
    m, o = both_meshes((2, 2, 2), 7)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    r = nk.FusedPCG(op, jac, tol=1e-8).solve(torch.zeros(m.n_local, dtype=torch.float64,
                                                        device="cuda"))
    assert r.iterations == 0 and r.converged and float(r.x.abs().max()) == 0.0
    # single element, all faces Dirichlet, N=1: every point is masked -> b = 0
    m1 = nk.build_box_mesh((1, 1, 1), (1, 1, 1), 1, bc="dirichlet")
    op1 = nk.PoissonOperator(m1)
    r1 = nk.pcg(op1, nk.JacobiPreconditioner(op1),
                torch.zeros(8, dtype=torch.float64, device="cuda"))
    assert r1.iterations == 0


@pytest.mark.parametrize("bc,lam1", [("dirichlet", 0.0), ("periodic", 2.0)])
def test_fused_pcg_order_one_element_per_thread(bc, lam1):
    """N = 1 runs the element-per-thread fused step (bk5_n1_pcg, the
    iterative coarse solve's kernel): iterations within +-1 of the oracle,
    same solution."""
    m, o = both_meshes((6, 5, 4), 1, bc=bc)
    op = nk.PoissonOperator(m, lam1=lam1)
    D, G = o.basis.diff, o.G
    mask = o.mask.ravel()
    sh = (o.G.shape[0],) + o.G.shape[2:]
    A = lambda v: mask * ogs.gs_op(o.ids, oop.bk5(D, G, v.reshape(sh), 1.0, o.B, lam1).ravel())
    inv = mask / ogs.gs_op(o.ids, oop.local_diagonal(D, G, 1.0, o.B, lam1).ravel())
    rng = np.random.default_rng(11)
    b = mask * ogs.gs_op(o.ids, rng.standard_normal(o.ids.size))
    ref = osol.pcg(A, lambda r: inv * r, b, tol=1e-9, max_iter=2000,
                   weights=1.0 / ogs.multiplicity(o.ids))
    res = nk.pcg(op, nk.JacobiPreconditioner(op), dev(b), tol=1e-9, max_iter=2000)
    assert res.converged and abs(res.iterations - ref.iterations) <= 1
    assert np.max(np.abs(res.x.cpu().numpy() - ref.x)) < 1e-7 * np.max(np.abs(ref.x))


def test_gs_handle_c_api_bit_exact():
    """nk_gs_create / nk_gs_apply / nk_gs_destroy (the library-owned handle a
    C caller uses): bit-exact against the oracle's canonical fold, including
    multiplicities > 32 (the CSR remainder) and more than 16 size classes."""
    import ctypes
    from paper_2104_05829_b200._lib import check, lib
    L = lib()
    rng = np.random.default_rng(7)
    ids = np.concatenate([np.repeat(np.arange(1, 200), 2), np.repeat(np.arange(200, 260), 3),
                          np.repeat([300], 40), np.repeat([301], 33),
                          np.concatenate([np.repeat(400 + k, k) for k in range(2, 26)]),
                          np.zeros(50, np.int64), np.arange(1000, 1100)]).astype(np.int64)
    ids = ids[rng.permutation(len(ids))]
    n = len(ids)
    perm = np.zeros(n, np.int32)
    seg = np.zeros(n // 2 + 2, np.int32)
    ns, npm = ctypes.c_int64(), ctypes.c_int64()
    check(L.nk_gs_plan_build(ids.ctypes.data, n, perm.ctypes.data, seg.ctypes.data,
                             ctypes.byref(ns), ctypes.byref(npm)), "plan")
    h = ctypes.c_void_p()
    check(L.nk_gs_create(perm.ctypes.data, seg.ctypes.data, ns.value, npm.value,
                         ctypes.byref(h)), "gs_create")
    try:
        for op in ("+", "min", "max", "*"):
            w = rng.standard_normal(n)
            wd = torch.as_tensor(w.copy(), device="cuda")
            from paper_2104_05829_b200._lib import OP_CODES
            check(L.nk_gs_apply(h, wd.data_ptr(), OP_CODES[op], 1, n, None,
                                torch.cuda.current_stream().cuda_stream), "gs_apply")
            assert np.array_equal(wd.cpu().numpy(), ogs.gs_op(ids, w, op)), op
    finally:
        check(L.nk_gs_destroy(h), "gs_destroy")


@pytest.mark.parametrize("op", ["+", "*", "min", "max"])
def test_gs_32bit_bit_exact(op):
    """SPEC.md:202 precision = 32-bit: float32 fields folded in FP32 in the
    canonical order -- bit-exact against the oracle's FP32 sequential fold."""
    m, o = both_meshes((3, 2, 2), 5, bc="periodic")
    h = nk.gs_setup(m.ids, nq=m.nq)
    rng = np.random.default_rng(3)
    w = rng.standard_normal(o.ids.size).astype(np.float32)
    if op == "*":
        w = (1.0 + 0.01 * w).astype(np.float32)
    got = nk.gs_op(h, torch.as_tensor(w, device="cuda"), op, precision=32).cpu().numpy()
    ref = ogs.gs_op(o.ids, w, op, precision=32)
    assert got.dtype == np.float32 and np.array_equal(got, ref)
    assert np.array_equal(nk.gs_op(h, w.copy(), op, precision=32), ref)     # numpy path
    with pytest.raises(nk.ContractError):
        nk.gs_op(h, torch.as_tensor(w, device="cuda"), op, precision=64)


@pytest.mark.parametrize("n_extra", [0, 1])
def test_cg_xpstep_unaligned_matches_vec(n_extra):
    """nk_cg_xpstep's scalar fallback (buffers offset by one double, not
    16-B aligned) against its 16-B path, bit for bit; n odd and even."""
    from paper_2104_05829_b200._lib import lib, ptr
    m, o = both_meshes((3, 3, 3), 2)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    rng = np.random.default_rng(3)
    b = torch.as_tensor(o.mask.ravel() * ogs.gs_op(o.ids, rng.standard_normal(m.n_local)),
                        device="cuda")
    s = nk.FusedPCG(op, jac, tol=1e-30, max_iter=3, split_step=True, use_graph=False, chunk=1)
    s.init(b)
    s._iteration()
    s._iteration()   # iter = 2: xpstep does the x and p updates
    n = s.n - n_extra
    L = lib()
    outs = []
    for off in (0, 1):
        buf = lambda v: torch.cat([torch.zeros(off, dtype=v.dtype, device="cuda"), v[:n]])
        x, r, p, d = buf(s.x), buf(s.r), buf(s.p), buf(s.invD)
        st = s.st.clone()
        sl = lambda t: t[off:]
        assert (sl(x).data_ptr() % 16 == 0) == (off == 0)
        _lib.check(L.nk_cg_xpstep(n, ptr(sl(x)), ptr(sl(r)), ptr(sl(p)), ptr(sl(d)), ptr(st),
                                  None, None), "xpstep")
        outs.append((sl(x).clone(), sl(p).clone()))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert not torch.equal(outs[0][0], s.x[:n])   # the update did run
