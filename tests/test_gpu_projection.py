"""GPU parity: projection-based initial guesses (paper_2104_05829_b200.projection,
libnekb200 nk_multi_wdot / nk_multi_axpy / nk_vscale) against
oracle/projection.py on the same mesh and right-hand sides.  Bars: projected
guess and deflated rhs within 1e-10 relative L2 (FP64, different summation
order), stored basis A-orthonormal to 1e-8, PCG iteration
counts within +-1 of the oracle, SPEC.md:535-537 examples."""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om
from oracle import operators as oop
from oracle import projection as oproj

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_05829_b200 as nk  # noqa: E402


def rel_l2(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", params=[(4, (2, 2, 2)), (7, (3, 3, 2))])
def setup(request):
    N, counts = request.param
    kw = dict(bc="dirichlet", deformation=("sine", 0.05))
    m = nk.build_box_mesh((1, 1, 1), counts, N, **kw)
    o = om.build_box_mesh((1, 1, 1), counts, N, **kw)
    op = nk.PoissonOperator(m)
    mask = o.mask.ravel()
    shape = (o.E,) + (N + 1,) * 3
    A = lambda v: mask * ogs.gs_op(o.ids, oop.bk5(o.basis.diff, o.G, v.reshape(shape)).ravel())
    inv = mask / ogs.gs_op(o.ids, oop.local_diagonal(o.basis.diff, o.G).ravel())
    wt = 1.0 / ogs.multiplicity(o.ids)
    rng = np.random.default_rng(2104_05829)
    rhs = [mask * ogs.gs_op(o.ids, o.B.ravel() * rng.standard_normal(mask.size))
           for _ in range(2)]
    b2 = rhs[0] + 0.01 * np.linalg.norm(rhs[0]) / np.linalg.norm(rhs[1]) * rhs[1]
    return dict(m=m, o=o, op=op, A=A, M=lambda r: inv * r, wt=wt, b=rhs[0], b2=b2, mask=mask)


def _rand(s, seed):
    o, mask = s["o"], s["mask"]
    x = np.random.default_rng(seed).standard_normal(mask.size)
    return mask * ogs.gs_op(o.ids, x / ogs.multiplicity(o.ids))


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def test_project_and_update_match_oracle(setup):
    s = setup
    sp = nk.ProjectionSpace(s["op"], capacity=3)
    osp = oproj.ProjectionSpace(3, s["wt"])
    x0, bd = sp.project(dev(s["b"]))
    assert not torch.any(x0) and torch.equal(bd, dev(s["b"]))
    for seed in range(5):                   # exercises eviction at capacity 3
        x = _rand(s, 20 + seed)
        sp.update(dev(x))                   # A x by the device operator
        osp.update(x, s["A"](x))
        assert sp.size == osp.size
        G = sp.gram()
        assert np.max(np.abs(G - np.eye(sp.size))) < 1e-8
        for q in range(sp.size):
            assert rel_l2(sp.X[q].cpu().numpy(), osp.X[q]) < 1e-9
        x0, bd = sp.project(dev(s["b"]))
        ox0, obd = osp.project(s["b"])
        assert rel_l2(x0.cpu().numpy(), ox0) < 1e-9
        assert rel_l2(bd.cpu().numpy(), obd) < 1e-9


def test_degenerate_restart(setup):
    s = setup
    sp = nk.ProjectionSpace(s["op"], capacity=8)
    x, y = _rand(s, 1), _rand(s, 2)
    sp.update(dev(y))
    sp.update(dev(x))
    assert sp.size == 2
    sp.update(dev(x))
    assert sp.size == 1 and sp.restarts == 1
    assert abs(sp.gram()[0, 0] - 1.0) < 1e-12


@pytest.mark.parametrize("solver_kind", ["jacobi", "pmg"])
def test_projected_solver_spec_examples(setup, solver_kind):
    s = setup
    op = s["op"]
    if solver_kind == "jacobi":
        solver = nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-8, max_iter=2000)
    else:
        solver = nk.MultigridPCG(op, tol=1e-8, max_iter=500)
    ps = nk.ProjectedSolver(solver, capacity=8)
    osp = oproj.ProjectionSpace(8, s["wt"])
    r1 = ps.solve(dev(s["b"]))
    x1 = r1.x.cpu().numpy().copy()
    r2 = ps.solve(dev(s["b"]))               # same rhs -> 0 iterations
    assert r2.iterations == 0 and r2.converged
    assert rel_l2(r2.x.cpu().numpy(), x1) < 1e-8
    r3 = ps.solve(dev(s["b2"]))              # 1% change -> fewer iterations
    assert r3.converged and r3.iterations < r1.iterations
    if solver_kind == "jacobi":
        o1 = oproj.solve_projected(osp, s["A"], s["M"], s["b"], tol=1e-8, max_iter=2000)
        oproj.solve_projected(osp, s["A"], s["M"], s["b"], tol=1e-8)
        o3 = oproj.solve_projected(osp, s["A"], s["M"], s["b2"], tol=1e-8, max_iter=2000)
        assert abs(r1.iterations - o1.iterations) <= 1
        assert abs(r3.iterations - o3.iterations) <= 1
        assert rel_l2(r3.x.cpu().numpy(), o3.x) < 1e-7
    # true residual of the projected answer meets the ORIGINAL tolerance
    res = dev(s["b2"]) - op(r3.x)
    wt = op.weights
    rn = float(torch.sqrt(torch.sum(wt * res * res)))
    bn = float(torch.sqrt(torch.sum(wt * dev(s["b2"]) ** 2)))
    assert rn <= 1e-7 * bn


def test_contract_errors(setup):
    s = setup
    with pytest.raises(nk.ContractError):
        nk.ProjectionSpace(s["op"], capacity=0)
    sp = nk.ProjectionSpace(s["op"], capacity=2)
    with pytest.raises(nk.ContractError):
        sp.project(torch.zeros(7, dtype=torch.float64, device="cuda"))
