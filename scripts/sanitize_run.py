"""Small end-to-end exercise of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2104_05829_b200 as nk
from paper_2104_05829_b200 import _lib

L = _lib.lib()
for N, counts in ((7, (3, 2, 2)), (4, (2, 2, 2)), (9, (2, 1, 1)), (12, (2, 1, 1))):
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    for v in (1, 3, 4):
        L.nk_bk5_set_variant(v)
        nk.apply_stiffness_local(u, m)
        nk.apply_stiffness_local(u, m, elements=torch.tensor([0, 2], dtype=torch.int32,
                                                             device="cuda"))
    L.nk_bk5_set_variant(0)
    u3 = torch.randn(3 * m.n_local, dtype=torch.float64, device="cuda")
    nk.apply_helmholtz_local(u3, m, 0.5, 2.0, ncomp=3)
    L.nk_bk5_set_variant(6)   # seq3: bk5_pencil<NC = 3>
    nk.apply_helmholtz_local(u3, m, 0.5, 2.0, ncomp=3)
    L.nk_bk5_set_variant(0)
    op = nk.PoissonOperator(m)
    jac = nk.JacobiPreconditioner(op)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    nk.FusedPCG(op, jac, tol=1e-6, max_iter=20, use_graph=False).solve(b)
    nk.pcg(lambda v: op(v), lambda r: jac(r), b, tol=1e-6, max_iter=10)
    uh = u.cpu().pin_memory()
    nk.apply_stiffness_local(uh, m)
torch.cuda.synchronize()
print("sanitize run ok")

# stage kernel (variant 8, bk5_stage.cuh): persistent CTAs that loop over
# several elements (u double buffer, G buffer, bulk w stores, the odd-NQ
# 8-byte phase shift and tail copy, the N = 15 tensor-map path), plain,
# Helmholtz + mask, the fused p.Ap of the split PCG step
for N, counts in ((8, (20, 20, 1)), (12, (15, 20, 1)), (12, (3, 3, 3)), (13, (10, 15, 2)),
                  (15, (10, 16, 2))):
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    L.nk_bk5_set_variant(8)
    nk.apply_stiffness_local(u, m)
    nk.apply_helmholtz_local(u, m, 0.5, 2.0)
    op = nk.PoissonOperator(m)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-6, max_iter=3, use_graph=False,
                split_step=True).solve(b)
    L.nk_bk5_set_variant(0)
torch.cuda.synchronize()
print("sanitize run (stage) ok")

# round-2 paths: the stage kernel with several elements per CTA (N = 6) and
# its alternative shapes (cfg 21 / 22: RINU, G4U at N = 14), the capped
# grid-stride fused-dot launches (pencil N = 3, 5; pencil2 N = 2; N = 1), the
# FDM on the FP64 tensor cores (N = 5, 9)
for N, counts, variant, cfg in ((6, (14, 14, 1), 8, 0), (14, (11, 11, 2), 8, 21),
                                (14, (11, 11, 2), 8, 22), (3, (40, 20, 1), 0, 0),
                                (5, (20, 20, 1), 0, 0), (2, (40, 40, 1), 0, 0),
                                (1, (60, 60, 2), 0, 0)):
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    L.nk_bk5_set_variant(variant)
    L.nk_bk5_tune(cfg, 1)
    nk.apply_stiffness_local(u, m)
    op = nk.PoissonOperator(m)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-6, max_iter=3, use_graph=False,
                split_step=True).solve(b)
    L.nk_bk5_set_variant(0)
    L.nk_bk5_tune(0, 1)
for N in (5, 9):
    m = nk.build_box_mesh((1, 1, 1), (3, 2, 2), N, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    r = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, r)
    for kind in ("asm", "ras"):
        L.nk_set_knob(3, 1)
        sm = nk.SchwarzSmoother(op, kind)
        z = torch.empty_like(r)
        sm.apply(r, z)
        L.nk_set_knob(3, 2)
torch.cuda.synchronize()
print("sanitize run (round-2 paths) ok")

# SURVEY.md §8f kernels: p-multigrid (interp3, cheb_step, dense matvec, the
# nested coarse PCG + cg_gate), Schwarz (fdm FP64/FP32, schwarz_post, ext gs),
# projection (multi_wdot, multi_axpy, vscale), the BK5 variant selection
for N, counts in ((5, (2, 2, 2)), (4, (3, 2, 1))):
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    op = nk.PoissonOperator(m)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    for sm, prec, coarse in (("cheby_jac", 64, "dense"), ("ras", 32, "pcg"),
                             ("cheby_asm", 64, "dense")):
        h = nk.MultigridHierarchy(op, smoother=sm, smoother_precision=prec, coarse=coarse,
                                  coarse_iters=5, power_iters=3)
        nk.MultigridPCG(op, h, tol=1e-6, max_iter=4, use_graph=False).solve(b)
    ps = nk.ProjectedSolver(nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-6,
                                        max_iter=30, use_graph=False), capacity=3)
    for s in range(4):
        ps.solve(b * (1.0 + 0.1 * s))
    nk.select_kernel_variant(m, reps=1)
    nk.kernels.reset_kernel_variant()
torch.cuda.synchronize()
print("sanitize run (pMG / Schwarz / projection) ok")

# late round-2 kernels: the single-buffer TMA BP5 step (N = 7, several
# elements per CTA), the pipelined gs update (grid-stride trips), the stage
# kernel with the fused PCG head (N = 8, 12), the N = 15 CTA-pair cluster
# kernel (variant 10: multicast u, st.async exchange), the N = 2 point kernel
# (variant 11, odd last group) and the stage16 kernel after the shared
# address-space fix
for N, counts, variant, split in ((7, (12, 12, 4), 0, False), (8, (10, 10, 3), 0, False),
                                  (12, (4, 4, 3), 0, False), (15, (5, 4, 3), 10, True),
                                  (15, (5, 4, 3), 8, True), (2, (7, 5, 3), 11, True)):
    m = nk.build_box_mesh((1, 1, 1), counts, N, deformation=("sine", 0.05))
    u = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    L.nk_bk5_set_variant(variant)
    nk.apply_stiffness_local(u, m)
    nk.apply_helmholtz_local(u, m, 0.5, 2.0)
    op = nk.PoissonOperator(m)
    b = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
    nk.gs_op(op.gs, b)
    b *= m.mask.reshape(-1).to(torch.float64)
    nk.FusedPCG(op, nk.JacobiPreconditioner(op), tol=1e-6, max_iter=4, use_graph=False,
                split_step=split).solve(b)
    L.nk_bk5_set_variant(0)
torch.cuda.synchronize()
print("sanitize run (late round-2 kernels) ok")
