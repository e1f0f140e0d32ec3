"""The edge / vertex gather-scatter folded into the persistent N = 7 BP5 step
(nk_bk5_pcg_gs, NK_KNOB_GS_TAIL): every CTA of the step meets a grid barrier
after its elements, then the >= 3-member segments are summed in the same lane
order and fold as nk_gs_op_classes.  The schedule is checked bit for bit
against the two-launch form (nk_bk5_pcg, then nk_gs_op_classes on the same
sub-plan), which test_gpu_parity / test_gpu_ring tie to the oracle -- at
sizes where each CTA takes one element (E = 64 < the 592-CTA grid) and where
the persistent grid cycles (E = 1000, the bench's E = 8000)."""

import numpy as np
import pytest

from oracle import gs as ogs
from oracle import mesh as om

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import _lib  # noqa: E402
from paper_2104_05829_b200.solvers import read_state  # noqa: E402

KNOB_GS_TAIL = 7


@pytest.fixture(autouse=True)
def tail_knob():
    """the tail is off by default (measured slower); these tests switch it on"""
    L = _lib.lib()
    old = L.nk_set_knob(KNOB_GS_TAIL, 1)
    yield
    L.nk_set_knob(KNOB_GS_TAIL, old)


def _rhs(m, o, seed):
    rng = np.random.default_rng(seed)
    return torch.as_tensor(o.mask.ravel() * ogs.gs_op(o.ids, rng.standard_normal(m.n_local)),
                           device="cuda")


@pytest.mark.parametrize("counts,bc,lam1,max_iter", [((4, 4, 4), "dirichlet", 0.0, 2000),
                                                     ((3, 4, 2), "periodic", 1.0, 2000),
                                                     ((3, 3, 3), "neumann", 0.5, 2000),
                                                     ((10, 10, 10), "dirichlet", 0.0, 2000),
                                                     ((20, 20, 20), "dirichlet", 0.0, 40)])
def test_gs_tail_solve_bit_identical(counts, bc, lam1, max_iter):
    """FusedPCG with the gs tail (2 launches per iteration) against the same
    solver with the separate gs pass (3 launches): same iterations, residual
    history and solution bit for bit, graph-replayed and eager."""
    N = 7
    m = nk.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc=bc, deformation=("sine", 0.05))
    o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc=bc, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m, lam1=lam1)
    jac = nk.JacobiPreconditioner(op)
    b = _rhs(m, o, 7)
    st = nk.FusedPCG(op, jac, tol=1e-9, max_iter=max_iter, split_step=False, gs_tail=True)
    assert st.gs_tail and st.launches_per_iter == 2
    sg = nk.FusedPCG(op, jac, tol=1e-9, max_iter=max_iter, split_step=False, gs_tail=False)
    assert not sg.gs_tail and sg.launches_per_iter == 3
    se = nk.FusedPCG(op, jac, tol=1e-9, max_iter=max_iter, split_step=False, gs_tail=True,
                     use_graph=False)
    rt, rg, re_ = st.solve(b), sg.solve(b), se.solve(b)
    assert rt.iterations == rg.iterations == re_.iterations
    assert rt.residual_history == rg.residual_history == re_.residual_history
    assert torch.equal(rt.x, rg.x) and torch.equal(rt.x, re_.x)
    if max_iter == 2000:
        assert rt.converged
        Ax = torch.empty_like(b)
        op(rt.x.reshape(-1), out=Ax)
        assert float(torch.linalg.norm(Ax - b)) <= 2e-9 * float(torch.linalg.norm(b))
    prof = st.profile_iteration(reps=2)
    assert set(prof) == {"bk5_pcg", "cg_update_gs"}


def test_bk5_pcg_gs_abi_one_step_matches_two_launches():
    """nk_bk5_pcg_gs through the C ABI, knob on (one launch, the tail) vs off
    (nk_bk5_pcg + nk_gs_op_classes): w, x, p and the state scalars after one
    step are bit-identical; the barrier's generation word advances once per
    fused launch and the arrival ticket is back at 0."""
    L = _lib.lib()
    N, counts = 7, (12, 10, 9)      # E = 1080: the persistent grid cycles
    m = nk.build_box_mesh((1.0, 1.0, 1.0), counts, N, deformation=("sine", 0.05))
    o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), split_step=False, use_graph=False)
    assert s.gs_tail
    s.init(_rhs(m, o, 3))
    # two iterations in so the step runs with beta != 0 and the deferred x update
    for _ in range(2):
        s._iteration()
    save = {k: getattr(s, k).clone() for k in ("x", "r", "p", "w", "st")}
    out = {}
    for knob in (1, 0):
        for k, v in save.items():
            getattr(s, k).copy_(v)
        L.nk_set_knob(KNOB_GS_TAIL, knob)
        assert L.nk_bk5_pcg_gs_fused(N) == knob
        s._step_gs_tail(L, _lib.stream_ptr())
        torch.cuda.synchronize()
        out[knob] = {k: getattr(s, k).clone() for k in ("x", "p", "w", "st")}
    for k in ("x", "p", "w"):
        assert torch.equal(out[1][k], out[0][k]), k
    st1, st0 = (read_state(out[q]["st"]) for q in (1, 0))
    assert st1.pAp == st0.pAp and st1.rz == st0.rz and st1.iter == st0.iter
    assert list(st1.ticket) == [0, 0, 0, 0] and list(st0.ticket) == [0, 0, 0, 0]
    assert st1.gen == read_state(save["st"]).gen + 1 and st0.gen == read_state(save["st"]).gen
    assert float(out[1]["w"].abs().sum()) > 0


def test_gs_tail_off_for_other_orders_and_ranks():
    """The tail is only offered where the step kernel is persistent (N = 7);
    elsewhere nk_bk5_pcg_gs runs the two launches and FusedPCG keeps the
    separate pass."""
    L = _lib.lib()
    assert L.nk_bk5_pcg_gs_fused(7) == 1
    for N in (3, 8, 12):
        assert L.nk_bk5_pcg_gs_fused(N) == 0
    m = nk.build_box_mesh((1.0, 1.0, 1.0), (3, 3, 3), 3, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    s = nk.FusedPCG(op, nk.JacobiPreconditioner(op), split_step=False, gs_tail=True)
    assert not s.gs_tail and s.launches_per_iter == 3


@pytest.mark.parametrize("counts,N,bc,lam1,split", [((4, 4, 4), 7, "dirichlet", 0.0, False),
                                                    ((10, 10, 10), 7, "periodic", 1.0, False),
                                                    ((20, 20, 20), 7, "dirichlet", 0.0, False),
                                                    ((5, 4, 3), 3, "neumann", 0.5, True),
                                                    ((6, 6, 6), 8, "dirichlet", 0.0, True)])
def test_gs_in_update_bit_identical(counts, N, bc, lam1, split):
    """NK_KNOB_GS_TAIL = 2: nk_cg_update_gs_cls runs the edge / vertex gs
    inside the update kernel before a grid barrier (one launch instead of
    two): same iterations, residual history and solution bit for bit as the
    separate passes (knob 0), graph-replayed, on the fused and split steps."""
    L = _lib.lib()
    m = nk.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc=bc, deformation=("sine", 0.05))
    o = om.build_box_mesh((1.0, 1.0, 1.0), counts, N, bc=bc, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m, lam1=lam1)
    jac = nk.JacobiPreconditioner(op)
    b = _rhs(m, o, 11)
    max_iter = 60 if m.E >= 8000 else 3000
    res = {}
    for knob in (2, 0):
        L.nk_set_knob(KNOB_GS_TAIL, knob)
        s = nk.FusedPCG(op, jac, tol=1e-9, max_iter=max_iter, split_step=split, gs_tail=False)
        assert s.launches_per_iter == (3 if split else 2) + (knob == 0)
        res[knob] = s.solve(b)
    assert res[2].iterations == res[0].iterations
    assert res[2].residual_history == res[0].residual_history
    assert torch.equal(res[2].x, res[0].x)
    if max_iter == 3000:
        assert res[2].converged
