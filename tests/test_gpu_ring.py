"""GPU parity at sizes where the persistent TMA kernels cycle their ring.

``bk5_pencil_tma`` (nk_bk5 variant 4) and ``bk5_pencil_tma_pcg`` (the fused
BP5 step at N = 7) launch ``min(E, 4 x 148 x ...)`` persistent CTAs
(csrc/bk5_tma.cuh); with E <= 64 every CTA processes one element and the
second ring stage, its mbarrier phase flip and the stage reuse never run.
These tests use E >= 1000 (E = 8000 is configs[1], the size the bench
times) so every CTA walks several elements through both stages.

Bars (BASELINE.json north_star): Ax within 1e-12 relative L2; PCG iterations
within +-1 of the oracle at the same tolerance.
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
from paper_2104_05829_b200 import kernels as K  # noqa: E402

BK5_TOL = 1e-12


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


class _OracleBP5:
    """Oracle BP5 problem on a box: b = mask QQ^T(B f), Jacobi, 1/mult dots;
    the gs plan is built once (oracle.gs.local_plan) and reused per apply."""

    def __init__(self, counts, N):
        o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc="dirichlet",
                              deformation=("sine", 0.05))
        self.o = o
        self.perm, self.seg = ogs.local_plan(o.ids)
        self.mask = o.mask.ravel()
        self.sh = (o.G.shape[0],) + o.G.shape[2:]
        X = o.xyz.reshape(3, -1)
        f = 3 * np.pi ** 2 * np.prod(np.sin(np.pi * X), axis=0)
        self.b = self.mask * self.gs(o.B.ravel() * f)
        D, G = o.basis.diff, o.G
        self.inv = self.mask / self.gs(oop.local_diagonal(D, G).ravel())
        self.wt = 1.0 / ogs.multiplicity(o.ids)

    def gs(self, v):
        return ogs.gs_op_plan(self.perm, self.seg, v).ravel()

    def A(self, v):
        o = self.o
        return self.mask * self.gs(oop.bk5(o.basis.diff, o.G, v.reshape(self.sh)).ravel())

    def residual(self, x):
        r = self.b - self.A(np.asarray(x).ravel())
        return float(np.sqrt(np.sum(self.wt * r * r)) / np.sqrt(np.sum(self.wt * self.b ** 2)))


@pytest.fixture
def variant_guard():
    L = _lib.lib()
    old = L.nk_bk5_set_variant(0)
    yield L
    L.nk_bk5_set_variant(old)


@pytest.mark.parametrize("counts", [(10, 10, 10), (20, 20, 20), (17, 13, 11)])
def test_bk5_tma_ring_reuse(variant_guard, counts):
    """nk_bk5 variant 4 (persistent pencil-TMA) vs the oracle at E = 1000,
    8000 (configs[1]) and a ragged E = 2431 (the last CTAs get one element
    fewer), plus an element subset longer than the grid."""
    N = 7
    L = variant_guard
    m = nk.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc="dirichlet", deformation=("sine", 0.05))
    o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc="dirichlet", deformation=("sine", 0.05))
    rng = np.random.default_rng(8000 + m.E)
    u = rng.standard_normal((m.E, 8, 8, 8))
    ref = oop.bk5(o.basis.diff, o.G, u)
    L.nk_bk5_set_variant(K.BK5_VARIANTS["pencil_tma"])
    w = nk.apply_stiffness_local(dev(u), m).cpu().numpy()
    assert rel_l2(w, ref) < BK5_TOL
    sub = rng.permutation(m.E)[: (m.E * 2) // 3].astype(np.int32)
    w2 = torch.full((m.E, 8, 8, 8), 3.0, dtype=torch.float64, device="cuda")
    nk.apply_stiffness_local(dev(u), m, out=w2, elements=dev(sub))
    w2 = w2.cpu().numpy()
    assert rel_l2(w2[sub], ref[sub]) < BK5_TOL
    rest = np.setdiff1d(np.arange(m.E), sub)
    assert np.all(w2[rest] == 3.0)
    # the pencil kernel (bench default) agrees with the TMA kernel to rounding
    L.nk_bk5_set_variant(K.BK5_VARIANTS["pencil"])
    w3 = nk.apply_stiffness_local(dev(u), m).cpu().numpy()
    assert rel_l2(w3, w) < BK5_TOL


def test_fused_tma_pcg_e1000_vs_oracle():
    """BP5 at N = 7 on a 10^3 box: the fused TMA step (bk5_pencil_tma_pcg,
    444 persistent CTAs for 1000 elements) against the oracle PCG --
    iterations +-1, x within 1e-7 (relative max)."""
    N = 7
    prob = _OracleBP5((10, 10, 10), N)
    ref = osol.pcg(prob.A, lambda r: prob.inv * r, prob.b, tol=1e-8, max_iter=2000,
                   weights=prob.wt)
    m = nk.build_box_mesh((1.0, 1.0, 1.0), (10, 10, 10), N, bc="dirichlet",
                          deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    s = nk.FusedPCG(op, jac, tol=1e-8, max_iter=2000)
    assert not s.split  # N = 7: the one-kernel TMA step
    res = s.solve(dev(prob.b))
    assert res.converged and ref.converged
    assert abs(res.iterations - ref.iterations) <= 1, (res.iterations, ref.iterations)
    x = res.x.cpu().numpy().ravel()
    assert np.max(np.abs(x - ref.x)) < 1e-7 * np.max(np.abs(ref.x))
    assert prob.residual(x) <= 1.05e-8
    # the split step (cg_xpstep + pencil BK5) lands on the same answer
    sp = nk.FusedPCG(op, jac, tol=1e-8, max_iter=2000, split_step=True)
    rs = sp.solve(dev(prob.b))
    assert abs(rs.iterations - ref.iterations) <= 1
    assert np.max(np.abs(rs.x.cpu().numpy().ravel() - ref.x)) < 1e-7 * np.max(np.abs(ref.x))


def test_fused_tma_pcg_config1_size():
    """configs[1] / configs[3] per-GPU size (E = 20^3, N = 7, the BP5 bench
    box): fused TMA step vs split (pencil) step -- same iterations (+-1) and
    x to 1e-9 relative; the oracle residual of the GPU solution meets the
    tolerance (one oracle apply at full size)."""
    N = 7
    prob = _OracleBP5((20, 20, 20), N)
    m = nk.build_box_mesh((1.0, 1.0, 1.0), (20, 20, 20), N, bc="dirichlet",
                          deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    b = dev(prob.b)
    fa = nk.FusedPCG(op, jac, tol=1e-8, max_iter=3000)
    fb = nk.FusedPCG(op, jac, tol=1e-8, max_iter=3000, split_step=True)
    ra, rb = fa.solve(b), fb.solve(b)
    assert ra.converged and rb.converged
    assert abs(ra.iterations - rb.iterations) <= 1
    xa = ra.x.cpu().numpy().ravel()
    xb = rb.x.cpu().numpy().ravel()
    assert np.max(np.abs(xa - xb)) < 1e-9 * np.max(np.abs(xa))
    assert prob.residual(xa) <= 1.05e-8
    # graph-replayed vs eager iterations: bit-identical
    fc = nk.FusedPCG(op, jac, tol=1e-8, max_iter=3000, use_graph=False, chunk=5)
    rc = fc.solve(b)
    assert rc.iterations == ra.iterations and torch.equal(rc.x, ra.x)


@pytest.mark.parametrize("counts", [(4, 4, 4), (10, 10, 10)])
def test_fused_tma_pcg_single_buffer_bit_identical(counts):
    """NK_KNOB_TMA = 1, 2 (single p / G buffers, five / four CTAs per SM) vs the
    two-stage ring (knob 0) at N = 7: only the copy schedule differs.  E = 64
    (one element per CTA, the same grid either way): bit-identical; E = 1000
    (every CTA cycles its buffers; 740 vs 444 CTAs, so the p.Ap partial sums
    are grouped differently): same iterations, x to 1e-12 relative.  With and
    without the PDL prologue."""
    L = _lib.lib()
    m = nk.build_box_mesh((1.0, 1.0, 1.0), counts, 7, bc="dirichlet",
                          deformation=("sine", 0.05))
    g = torch.Generator(device="cuda").manual_seed(3)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda", generator=g)
    op = nk.PoissonOperator(m)
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    jac = nk.JacobiPreconditioner(op)
    out = []
    old_pdl = L.nk_set_knob(0, 5)
    try:
        for pdl in (5, 0):
            L.nk_set_knob(0, pdl)
            for tma in (0, 1, 2):
                old = L.nk_set_knob(4, tma)
                try:
                    s = nk.FusedPCG(op, jac, tol=1e-8, max_iter=3000, chunk=16)
                    assert not s.split
                    out.append(s.solve(b))
                finally:
                    L.nk_set_knob(4, old)
    finally:
        L.nk_set_knob(0, old_pdl)
    assert out[0].converged
    same_grid = m.E <= 444
    for r in out[1:]:
        assert r.iterations == out[0].iterations
        if same_grid:
            assert torch.equal(r.x, out[0].x)
        else:
            assert float((r.x - out[0].x).abs().max()) <= 1e-12 * float(out[0].x.abs().max())


@pytest.mark.parametrize("counts,N", [((3, 3, 3), 5), ((10, 10, 10), 7), ((20, 20, 20), 7)])
def test_cg_update_gs_pipelined_bit_identical(counts, N):
    """NK_KNOB_CG_PIPE = 1, 2 (nk_cg_update_gs software-pipelined one / two
    deep across its grid-stride trips) vs 0: same per-thread point order and accumulation,
    so the converged fused-gs solve is bit-identical -- at E = 8000 every
    thread runs ~7 trips, so the carried registers are exercised."""
    L = _lib.lib()
    m = nk.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc="dirichlet",
                          deformation=("sine", 0.05))
    g = torch.Generator(device="cuda").manual_seed(5)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda", generator=g)
    op = nk.PoissonOperator(m)
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    jac = nk.JacobiPreconditioner(op)
    out = []
    for pipe in (4, 5, 6):   # the 4 x 148-block grid; pipelining 0 / 1 / 2
        old = L.nk_set_knob(5, pipe)
        try:
            s = nk.FusedPCG(op, jac, tol=1e-8, max_iter=3000, chunk=16, split_step=False)
            assert s.codes is not None
            out.append(s.solve(b))
        finally:
            L.nk_set_knob(5, old)
    assert out[0].converged
    for o in out[1:]:
        assert o.iterations == out[0].iterations
        assert o.residual_history == out[0].residual_history
        assert torch.equal(o.x, out[0].x)


@pytest.mark.parametrize("N,counts", [(8, (3, 3, 3)), (8, (10, 10, 10)), (9, (4, 3, 3)),
                                      (10, (3, 3, 2)), (11, (3, 3, 3)), (12, (3, 2, 2)),
                                      (13, (2, 2, 3)), (14, (3, 3, 3))])
def test_stage_pcg_step_matches_split(N, counts):
    """nk_bk5_pcg on the stage kernel with the PCG head fused into its F3
    pass (N + 1 in 9..15, NK_KNOB_STAGE_PCG) against the split step
    (nk_cg_xpstep + the stage BK5 with the fused p.Ap): the same per-point
    arithmetic and the same partial-sum grouping, so iterations, residual
    history and x are bit-identical; E = 1000 at N = 8 cycles every CTA's
    buffers several times."""
    m = nk.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc="dirichlet",
                          deformation=("sine", 0.05))
    g = torch.Generator(device="cuda").manual_seed(9)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda", generator=g)
    op = nk.PoissonOperator(m)
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    jac = nk.JacobiPreconditioner(op)
    fused = nk.FusedPCG(op, jac, tol=1e-8, max_iter=3000, chunk=16, split_step=False)
    split = nk.FusedPCG(op, jac, tol=1e-8, max_iter=3000, chunk=16, split_step=True)
    rf, rs = fused.solve(b), split.solve(b)
    assert rf.converged and rf.iterations == rs.iterations
    assert rf.residual_history == rs.residual_history
    assert torch.equal(rf.x, rs.x)
    Ax = torch.empty_like(b)
    op(rf.x.reshape(-1), out=Ax)
    assert float(torch.linalg.norm(Ax - b)) <= 2e-8 * float(torch.linalg.norm(b))
