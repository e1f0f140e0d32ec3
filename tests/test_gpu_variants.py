"""GPU: select_kernel_variant -- measured BK5 variant
choice with deterministic tie-break, forced override, eligibility, and every
variant agreeing with the oracle to 1e-12."""

import numpy as np
import pytest

from oracle import mesh as om
from oracle import operators as oop

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import kernels as K  # noqa: E402


@pytest.mark.parametrize("N", [2, 3, 7, 12])
def test_select_variant_and_parity(N):
    counts = (3, 2, 2)
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    o = om.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = np.random.default_rng(N).standard_normal((m.E,) + (N + 1,) * 3)
    ref = oop.bk5(o.basis.diff, o.G, u)
    try:
        chosen = nk.select_kernel_variant(m, reps=5)
        assert K.bk5_variant_eligible(chosen, N)
        rep = K.variant_report()[-1]
        assert rep["chosen"] == chosen and not rep["forced"]
        assert set(rep["median_ms"]) == {v for v in K.BK5_VARIANTS if K.bk5_variant_eligible(v, N)}
        for v in K.BK5_VARIANTS:
            if not K.bk5_variant_eligible(v, N):
                continue
            assert nk.select_kernel_variant(m, candidates=[v], reps=1) == v   # one candidate
            w = nk.apply_stiffness_local(torch.as_tensor(u, device="cuda"), m).cpu().numpy()
            assert np.linalg.norm(w - ref) / np.linalg.norm(ref) < 1e-12, v
        assert nk.select_kernel_variant(m, force="kslab") == "kslab"
        assert K.variant_report()[-1]["forced"]
    finally:
        K.reset_kernel_variant()


def test_variant_errors():
    m = nk.build_box_mesh((1, 1, 1), (1, 1, 1), 5)
    with pytest.raises(nk.ContractError):
        nk.select_kernel_variant(m, candidates=["full3d"])
    m9 = nk.build_box_mesh((1, 1, 1), (1, 1, 1), 9)
    with pytest.raises(nk.ContractError):                  # N+1 = 10: TMA not eligible
        nk.select_kernel_variant(m9, candidates=["pencil_tma"], reps=1)
    with pytest.raises(nk.ContractError):
        nk.select_kernel_variant(m, force="bogus")
