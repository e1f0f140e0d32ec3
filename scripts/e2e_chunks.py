"""e2e host-buffer BK5 (apply_stiffness_local on pinned host u/w) vs chunk
count, next to the concurrent H2D+D2H floor of the same bytes."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05829_b200 as nk
m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
n = m.n_local
uh = torch.randn(n, dtype=torch.float64).pin_memory()
wh = torch.empty(n, dtype=torch.float64).pin_memory()


def t(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    mm = torch.cuda.current_stream()
    s1.wait_stream(mm)
    s2.wait_stream(mm)
    with torch.cuda.stream(s1):
        d1.copy_(uh, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    mm.wait_stream(s1)
    mm.wait_stream(s2)


out = {"floor_both_ms": round(t(both), 4),
       "h2d_ms": round(t(lambda: d1.copy_(uh, non_blocking=True)), 4),
       "d2h_ms": round(t(lambda: h2.copy_(d2, non_blocking=True)), 4)}
for k in (2, 4, 6, 8, 12, 16, 24, 32):
    out[f"e2e_ms_{k}"] = round(t(lambda: nk.apply_stiffness_local(uh, m, out=wh, nchunks=k)), 4)
print(json.dumps(out))

# zero-copy: the BK5 kernel reads u from and writes w to pinned host memory
# directly (UVA device-accessible addresses), no staging copies
from paper_2104_05829_b200._lib import check, lib, ptr  # noqa: E402
L = lib()


def zc():
    check(L.nk_bk5(m.N, m.E, ptr(m.basis.diff), ptr(m.G), uh.data_ptr(), wh.data_ptr(), 1.0,
                   None, 0.0, 1, n, None, None, 0, None, None, 0, 0,
                   torch.cuda.current_stream().cuda_stream), "bk5")


wd = torch.empty(n, dtype=torch.float64, device="cuda")
ref = nk.apply_stiffness_local(uh.cuda(), m, out=wd).cpu()
zc()
torch.cuda.synchronize()
out2 = {"zero_copy_ms": round(t(zc), 4), "zero_copy_equal": bool(torch.equal(wh, ref))}
for v in (3, 5, 1, 8):
    old = L.nk_bk5_set_variant(v)
    out2[f"zero_copy_ms_variant{v}"] = round(t(zc), 4)
    if v == 8:   # stage: TMA bulk loads of u from and bulk stores of w to pinned host memory
        wh.zero_()
        zc()
        torch.cuda.synchronize()
        out2["zero_copy_variant8_bitwise"] = bool(torch.equal(wh, ref))
    L.nk_bk5_set_variant(old)
print(json.dumps(out2))

# hybrid: copy-engine H2D per chunk, the chunk's BK5 writes w straight to
# pinned host memory (no D2H copies, no copy-out tail)
nq3 = m.nq ** 3
s_in, s_cmp = torch.cuda.Stream(), torch.cuda.Stream()
ud = torch.empty(n, dtype=torch.float64, device="cuda")


def hybrid(k):
    E = m.E
    b = [round(E * i / k) for i in range(k + 1)]
    mm = torch.cuda.current_stream()
    s_in.wait_stream(mm)
    for c in range(k):
        a0, a1 = b[c] * nq3, b[c + 1] * nq3
        with torch.cuda.stream(s_in):
            ud[a0:a1].copy_(uh[a0:a1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
        s_cmp.wait_event(ev)
        ne = b[c + 1] - b[c]
        check(L.nk_bk5(m.N, ne, ptr(m.basis.diff), m.G.data_ptr() + b[c] * 6 * nq3 * 8,
                       ud.data_ptr() + a0 * 8, wh.data_ptr() + a0 * 8, 1.0, None, 0.0, 1,
                       ne * nq3, None, None, 0, None, None, 0, 0, s_cmp.cuda_stream), "bk5")
    mm.wait_stream(s_cmp)


out3 = {}
for v in (0, 1, 8):
    old = L.nk_bk5_set_variant(v)
    for k in (2, 4, 6, 8, 12, 16):
        out3[f"hybrid_v{v}_k{k}"] = round(t(lambda: hybrid(k)), 4)
    if v == 8:   # the stage kernel's bulk stores (cp.async.bulk) into pinned host memory
        hybrid(8)
        torch.cuda.synchronize()
        out3["hybrid_v8_equal"] = bool(torch.allclose(wh, ref, rtol=1e-12, atol=0))
        out3["hybrid_v8_bitwise"] = bool(torch.equal(wh, ref))
    L.nk_bk5_set_variant(old)
hybrid(8)
torch.cuda.synchronize()
out3["hybrid_equal"] = bool(torch.equal(wh, ref))
print(json.dumps(out3))
