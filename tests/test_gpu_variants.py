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


@pytest.mark.parametrize("N", [2, 3, 7, 8, 12, 15])
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


@pytest.mark.parametrize("variant,N,counts", [
    (7, 8, (3, 2, 2)), (7, 9, (2, 2, 3)), (7, 12, (3, 2, 2)), (7, 13, (2, 3, 1)),
    (7, 14, (2, 2, 2)), (7, 15, (3, 2, 2)),
    (8, 2, (3, 2, 2)), (8, 4, (3, 3, 3)), (8, 5, (3, 2, 2)), (8, 6, (3, 3, 1)),
    (8, 7, (3, 2, 2)), (8, 8, (3, 3, 3)), (8, 9, (3, 2, 2)), (8, 10, (2, 2, 3)), (8, 11, (3, 3, 3)), (8, 12, (3, 3, 3)),
    (8, 13, (2, 3, 1)), (8, 14, (3, 3, 1)), (8, 15, (3, 2, 3)),
    (9, 8, (3, 3, 3)), (9, 9, (2, 2, 3)), (9, 11, (3, 2, 2)), (9, 12, (3, 3, 3)),
    (9, 13, (2, 3, 1)), (9, 14, (3, 3, 1)),
    (10, 15, (3, 3, 3)), (10, 15, (1, 1, 1)), (10, 15, (7, 6, 5)),
    (11, 2, (3, 2, 2)), (11, 2, (7, 5, 3)), (11, 2, (30, 30, 30))])
def test_dmma_variant_parity_fused(variant, N, counts):
    """Variant 7 (FP64 tensor-core contractions, bk5_dmma.cuh) and variant 8
    (TMA-staged operands, bk5_stage.cuh): persistent CTAs that each take
    several elements.  w vs the oracle with the Helmholtz mass term and the
    Dirichlet mask, and the fused p.Ap (nk_bk5 with a CG state) vs the host
    dot, at every order they serve; odd E at odd N + 1 (27 elements at
    N = 12) exercises the stage kernel's last-double tail copy."""
    from paper_2104_05829_b200._lib import check, lib, ptr
    from oracle import gs as ogs  # noqa: F401
    L = lib()
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    o = om.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = np.random.default_rng(100 + N).standard_normal((m.E,) + (N + 1,) * 3)
    lam0, lam1 = 0.7, 2.5
    ref = lam0 * oop.bk5(o.basis.diff, o.G, u) + lam1 * o.B * u
    ref = ref * o.mask
    old = L.nk_bk5_set_variant(variant)
    try:
        ut = torch.as_tensor(u, device="cuda").reshape(-1)
        w = torch.empty_like(ut)
        st = torch.zeros(256, dtype=torch.uint8, device="cuda")
        nb = int(L.nk_bk5_blocks(N, m.E, 1))
        assert 1 <= nb <= (2 if variant == 10 else 1) * m.E
        part = torch.zeros(nb, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        check(L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), ptr(ut), ptr(w), lam0, ptr(m.B),
                       lam1, 1, m.n_local, ptr(m.mask), None, 0, ptr(st), ptr(part), 0, nb, s),
              "bk5")
        wh = w.cpu().numpy().reshape(ref.shape)
        assert np.linalg.norm(wh - ref) / np.linalg.norm(ref) < 1e-12
        pap = float(st[8:16].view(torch.float64).item())
        assert abs(pap - float(np.sum(u * ref))) <= 1e-11 * abs(float(np.sum(u * ref)))
    finally:
        L.nk_bk5_set_variant(old)


@pytest.mark.parametrize("N,counts", [(2, (30, 30, 30)), (4, (16, 16, 16)), (6, (12, 12, 12)),
                                      (8, (12, 12, 12)), (9, (10, 10, 10)), (12, (10, 10, 10)),
                                      (13, (9, 9, 9)), (15, (7, 7, 7)),
                                      (14, (8, 8, 8))])
@pytest.mark.parametrize("variant", [8, 9])
def test_stage_variant_ring_reuse(N, counts, variant):
    """Variants 8 and 9 at sizes where every persistent CTA takes several elements
    (E >> 148 x CTAs per SM): the u / G buffers and both mbarrier phases are
    reused many times.  The contractions and their order are pencil2's, so
    w is bit-identical to variant 5, and within 1e-12 of the oracle."""
    from paper_2104_05829_b200._lib import lib
    L = lib()
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    o = om.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = np.random.default_rng(7 + N).standard_normal((m.E,) + (N + 1,) * 3)
    ref = oop.bk5(o.basis.diff, o.G, u)
    ut = torch.as_tensor(u, device="cuda")
    if variant == 9 and not 9 <= N + 1 <= 15:
        pytest.skip("stage2 serves N + 1 in 9..15")
    old = L.nk_bk5_set_variant(variant)
    try:
        w8 = nk.apply_stiffness_local(ut, m)
        L.nk_bk5_set_variant(5)
        w5 = nk.apply_stiffness_local(ut, m)
    finally:
        L.nk_bk5_set_variant(old)
    assert torch.equal(w8, w5)
    wh = w8.cpu().numpy()
    assert np.linalg.norm(wh - ref) / np.linalg.norm(ref) < 1e-12


@pytest.mark.parametrize("N", [12, 13])
def test_stage_variant_misaligned_slice(N):
    """u as an 8-byte-offset slice: the bulk copies start one double early
    (odd N + 1: every other element; even N + 1: every element, with the
    16-byte row reads falling back to 8-byte ones).  (N = 15's tensor-map
    staging needs 16-byte alignment and reports an error instead.)"""
    from paper_2104_05829_b200._lib import check, lib, ptr
    L = lib()
    counts = (3, 2, 3)
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    o = om.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = np.random.default_rng(3 + N).standard_normal((m.E,) + (N + 1,) * 3)
    ref = oop.bk5(o.basis.diff, o.G, u)
    buf = torch.zeros(m.n_local + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.as_tensor(u.reshape(-1), device="cuda")
    w = torch.empty(m.n_local, dtype=torch.float64, device="cuda")
    old = L.nk_bk5_set_variant(8)
    try:
        check(L.nk_bk5(N, m.E, ptr(m.basis.diff), ptr(m.G), buf.data_ptr() + 8, ptr(w), 1.0,
                       None, 0.0, 1, m.n_local, None, None, 0, None, None, 0, 0,
                       torch.cuda.current_stream().cuda_stream), "bk5")
    finally:
        L.nk_bk5_set_variant(old)
    wh = w.cpu().numpy().reshape(ref.shape)
    assert np.linalg.norm(wh - ref) / np.linalg.norm(ref) < 1e-12


@pytest.mark.parametrize("N", [4, 6, 12])
def test_stage_variant_element_subset(N):
    """Variant 8 over an element list (the multi-rank boundary / interior
    split): odd-length, unordered subsets -- several elements per CTA at the
    low orders with a partial last group -- vs the oracle on those elements
    (elements outside the list are not written)."""
    from paper_2104_05829_b200._lib import lib
    L = lib()
    counts = (5, 4, 3)
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    o = om.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = np.random.default_rng(11 + N).standard_normal((m.E,) + (N + 1,) * 3)
    ref = oop.bk5(o.basis.diff, o.G, u)
    sel = np.random.default_rng(N).permutation(m.E)[:37].astype(np.int32)
    old = L.nk_bk5_set_variant(8)
    try:
        w = nk.apply_stiffness_local(torch.as_tensor(u, device="cuda"), m,
                                     elements=torch.as_tensor(sel, device="cuda"))
    finally:
        L.nk_bk5_set_variant(old)
    wh = w.cpu().numpy().reshape(ref.shape)
    assert np.linalg.norm(wh[sel] - ref[sel]) / np.linalg.norm(ref[sel]) < 1e-12


@pytest.mark.parametrize("counts,subset", [((7, 7, 7), 0), ((9, 9, 9), 0), ((5, 4, 3), 37)])
def test_pair_variant_ring_and_subset(counts, subset):
    """Variant 10 (one N = 15 element per CTA pair, bk5_pair.cuh): E = 343 /
    729 (every cluster cycles its u / G / exchange buffers and both mbarrier
    phases several times) and an odd, unordered element subset -- vs the
    oracle at 1e-12, and vs variant 5 (pencil2) to rounding."""
    from paper_2104_05829_b200._lib import lib
    L = lib()
    N = 15
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    o = om.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = np.random.default_rng(17).standard_normal((m.E,) + (N + 1,) * 3)
    ref = oop.bk5(o.basis.diff, o.G, u)
    ut = torch.as_tensor(u, device="cuda")
    sel = (np.random.default_rng(1).permutation(m.E)[:subset].astype(np.int32)
           if subset else np.arange(m.E, dtype=np.int32))
    kw = {"elements": torch.as_tensor(sel, device="cuda")} if subset else {}
    old = L.nk_bk5_set_variant(10)
    try:
        w10 = nk.apply_stiffness_local(ut, m, **kw)
        L.nk_bk5_set_variant(5)
        w5 = nk.apply_stiffness_local(ut, m, **kw)
    finally:
        L.nk_bk5_set_variant(old)
    a10 = w10.cpu().numpy().reshape(ref.shape)[sel]
    a5 = w5.cpu().numpy().reshape(ref.shape)[sel]
    assert np.linalg.norm(a10 - ref[sel]) / np.linalg.norm(ref[sel]) < 1e-12
    assert np.linalg.norm(a10 - a5) / np.linalg.norm(a5) < 1e-13


def test_variant_errors():
    m = nk.build_box_mesh((1, 1, 1), (1, 1, 1), 5)
    with pytest.raises(nk.ContractError):
        nk.select_kernel_variant(m, candidates=["full3d"])
    m9 = nk.build_box_mesh((1, 1, 1), (1, 1, 1), 9)
    with pytest.raises(nk.ContractError):                  # N+1 = 10: TMA not eligible
        nk.select_kernel_variant(m9, candidates=["pencil_tma"], reps=1)
    with pytest.raises(nk.ContractError):
        nk.select_kernel_variant(m, force="bogus")
