"""The stage BK5 kernel reading u from / writing w to pinned host memory (UVA) vs
device buffers, next to the plain copy-engine H2D / D2H of the same bytes."""
import os, sys, json, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_2104_05829_b200 as nk
from paper_2104_05829_b200._lib import lib, ptr, check
L = lib()
m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
n = m.n_local
ud = torch.randn(n, dtype=torch.float64, device="cuda")
wd = torch.empty_like(ud)
wh = torch.empty(n, dtype=torch.float64).pin_memory()
uh = ud.cpu().pin_memory()
s = torch.cuda.current_stream().cuda_stream
def run(u, w, v):
    old = L.nk_bk5_set_variant(v)
    check(L.nk_bk5(7, m.E, ptr(m.basis.diff), ptr(m.G), u, w, 1.0, None, 0.0, 1, n, None, None, 0, None, None, 0, 0, s), "bk5")
    L.nk_bk5_set_variant(old)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps, 4)
out = {}
out["stage_dev_dev"] = t(lambda: run(ud.data_ptr(), wd.data_ptr(), 8))
out["stage_dev_to_host"] = t(lambda: run(ud.data_ptr(), wh.data_ptr(), 8))
out["stage_host_to_dev"] = t(lambda: run(uh.data_ptr(), wd.data_ptr(), 8))
out["stage_host_host"] = t(lambda: run(uh.data_ptr(), wh.data_ptr(), 8))
out["copy_d2h"] = t(lambda: wh.copy_(wd, non_blocking=True))
out["copy_h2d"] = t(lambda: ud.copy_(uh, non_blocking=True))
print(json.dumps(out))
