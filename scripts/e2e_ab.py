"""A/B of the host-buffer e2e apply (bench.py's protocol: L2 flushed, then
apply_stiffness_local on pinned host u / w, CUDA events around the call):
the copy pipeline (H2D / BK5 / D2H) vs the direct mode (H2D + stage-kernel
bulk stores into host memory, one kernel per chunk) vs the stream mode (one
chunk-gated stage kernel over all chunks), alternating in one process."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05829_b200 as nk  # noqa: E402
from paper_2104_05829_b200 import kernels as K  # noqa: E402
from paper_2104_05829_b200._lib import lib, ptr  # noqa: E402

L = lib()
m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
n = m.n_local
uh = torch.randn(n, dtype=torch.float64).pin_memory()
wh = torch.empty(n, dtype=torch.float64).pin_memory()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
res = {}
for rnd in range(4):
    for mode, orders, stream in (("copy", (), False), ("direct", (7,), False),
                                 ("stream", (7,), True)):
        for nch in ((6, 8) if mode != "stream" else (8, 16, 32)):
            K._HostStream.DIRECT_ORDERS = orders
            K._HostStream.STREAM = stream
            m._host_stream = None
            for _ in range(3):
                nk.apply_stiffness_local(uh, m, out=wh, nchunks=nch)
            ts = []
            for _ in range(60):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                L.nk_l2_flush(ptr(flush), flush.numel(), s.cuda_stream)
                a.record(s)
                nk.apply_stiffness_local(uh, m, out=wh, nchunks=nch)
                b.record(s)
                ts.append((a, b))
            torch.cuda.synchronize()
            res.setdefault(f"{mode}_k{nch}", []).append(
                round(statistics.mean([a.elapsed_time(b) for a, b in ts]), 4))
print(json.dumps(res))
