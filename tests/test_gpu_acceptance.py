"""SPEC.md acceptance criteria that fall on the hot path, run through the
product on the GPU:

* acceptance 1: spectral convergence of the BP5 solve;
* SPD: u^T A u > 0 for 100 random masked u;
* acceptance 10 / SPEC.md:433, 773: KernelCounters totals equal the closed
  forms exactly, per invocation, for every public entry point that applies
  the stiffness operator (device and host fields, element subsets, the
  3-component batch, the operator, the fused and multigrid PCG solves);
* acceptance 12: determinism (byte-identical results).
"""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200.kernels import COUNTERS, bk5_flops  # noqa: E402


def _manufactured(N, counts=(2, 2, 2), deformation=None):
    m = nk.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc="dirichlet", deformation=deformation)
    o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc="dirichlet", deformation=deformation)
    X = o.xyz.reshape(3, -1)
    ue = np.prod(np.sin(np.pi * X), axis=0)
    b = o.mask.ravel() * ogs.gs_op(o.ids, o.B.ravel() * 3 * np.pi ** 2 * ue)
    return m, ue, torch.as_tensor(b, device="cuda")


def test_spectral_convergence_acceptance_1():
    """Poisson, manufactured u = sin(pi x) sin(pi y) sin(pi z), E = 8
    Dirichlet box: for N = 2, 4, 6, 8, 10 the max-norm error decreases
    monotonically and by >= 10x per step of 2 until it reaches <= 1e-10."""
    errs = []
    for N in (2, 4, 6, 8, 10):
        m, ue, b = _manufactured(N)
        op = nk.PoissonOperator(m)
        res = nk.pcg(op, nk.JacobiPreconditioner(op), b, tol=1e-13, max_iter=2000)
        assert res.converged
        errs.append(float(np.max(np.abs(res.x.cpu().numpy().ravel() - ue))))
    for a, c in zip(errs, errs[1:]):
        if a <= 1e-10:
            break
        assert c < a and c <= a / 10.0, errs
    assert min(errs) <= 1e-10, errs


def test_spd_random_masked_vectors():
    """u^T A u > 0 for 100 random nonzero masked u (assembled,
    Dirichlet-masked stiffness on a deformed mesh)."""
    m = nk.build_box_mesh((1.0, 1.0, 1.0), (3, 2, 2), 5, bc="dirichlet",
                          deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    mask = m.mask.reshape(-1).to(torch.float64)
    wt = op.weights
    g = torch.Generator(device="cuda").manual_seed(432)
    vals = []
    for _ in range(100):
        u = torch.randn(m.n_local, dtype=torch.float64, device="cuda", generator=g)
        nk.gs_op(op.gs, u)            # continuous (assembled) field ...
        u *= mask                     # ... in the masked subspace
        Au = op(u)
        vals.append(float(torch.sum(wt * u * Au)))
    assert min(vals) > 0.0


@pytest.mark.parametrize("N", [3, 7, 10])
def test_kernel_counters_exact(N):
    """Counter totals match 12E(N+1)^4 + 15E(N+1)^3 flops and 7E(N+1)^3
    memory references per stiffness application, exactly."""
    nq = N + 1
    m = nk.build_box_mesh((1.0, 1.0, 1.0), (3, 2, 2), N, bc="dirichlet",
                          deformation=("sine", 0.05))
    E = m.E
    per = 12 * E * nq ** 4 + 15 * E * nq ** 3
    refs = 7 * E * nq ** 3
    assert bk5_flops(N, E) == per
    u = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    COUNTERS.reset()
    nk.apply_stiffness_local(u, m)
    assert COUNTERS.flops == {"stiffness": per} and COUNTERS.memory_refs == {"stiffness": refs}
    # host (pinned) field through the chunked pipeline, twice (graph replay)
    uh = u.cpu().pin_memory()
    nk.apply_stiffness_local(uh, m)
    nk.apply_stiffness_local(uh, m)
    assert COUNTERS.flops["stiffness"] == 3 * per
    # element subset: counted for the elements applied
    sub = torch.tensor([0, 2, 5], dtype=torch.int32, device="cuda")
    nk.apply_stiffness_local(u, m, out=torch.zeros_like(u), elements=sub)
    assert COUNTERS.flops["stiffness"] == 3 * per + 3 * (12 * nq ** 4 + 15 * nq ** 3)
    # 3-component Helmholtz batch: three applications
    COUNTERS.reset()
    nk.apply_helmholtz_local(torch.randn(3 * m.n_local, dtype=torch.float64, device="cuda"), m,
                             0.5, 2.0, ncomp=3)
    assert COUNTERS.flops == {"stiffness": 3 * per}
    assert COUNTERS.memory_refs == {"stiffness": 3 * refs}
    # the assembled operator: one application per call
    op = nk.PoissonOperator(m)
    COUNTERS.reset()
    op(u)
    op(u)
    assert COUNTERS.flops == {"stiffness": 2 * per}
    # fused PCG (graph-captured, chunked): one application per iteration
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    jac = nk.JacobiPreconditioner(op)
    for split in (False, True):
        s = nk.FusedPCG(op, jac, tol=1e-8, max_iter=500, chunk=7, split_step=split)
        COUNTERS.reset()
        r1 = s.solve(b)
        r2 = s.solve(b)          # replay of the captured chunk
        assert COUNTERS.flops == {"stiffness": (r1.iterations + r2.iterations) * per}
        assert COUNTERS.memory_refs == {"stiffness": (r1.iterations + r2.iterations) * refs}


def test_kernel_counters_multigrid_per_iteration():
    """MultigridPCG: the counts of a solve are (counts of the init V-cycle)
    + iterations x (counts of one iteration) -- identical for the first solve
    (with the graph capture) and a replayed second solve."""
    m = nk.build_box_mesh((1.0, 1.0, 1.0), (3, 3, 2), 6, bc="dirichlet",
                          deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    s = nk.MultigridPCG(op, nk.MultigridHierarchy(op), tol=1e-8, max_iter=100)
    COUNTERS.reset()
    r1 = s.solve(b)
    c1 = COUNTERS.flops["stiffness"]
    COUNTERS.reset()
    r2 = s.solve(b)
    c2 = COUNTERS.flops["stiffness"]
    assert r1.iterations == r2.iterations and c1 == c2 > 0
    # the fine level contributes one outer A p per iteration at least
    assert c1 >= r1.iterations * bk5_flops(6, m.E)


def test_determinism_acceptance_12():
    """Two runs of the same solve produce byte-identical results."""
    m, ue, b = _manufactured(7, counts=(3, 3, 3), deformation=("sine", 0.05))
    out = []
    for _ in range(2):
        op = nk.PoissonOperator(m)
        res = nk.pcg(op, nk.JacobiPreconditioner(op), b, tol=1e-10, max_iter=2000)
        mg = nk.MultigridPCG(op, nk.MultigridHierarchy(op, smoother="ras"), tol=1e-10,
                             max_iter=100).solve(b)
        out.append((res.x.cpu().numpy().tobytes(), tuple(res.residual_history),
                    mg.x.cpu().numpy().tobytes(), tuple(mg.residual_history)))
    assert out[0] == out[1]
