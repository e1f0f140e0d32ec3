"""e2e host-path chunk sweep (apply_stiffness_local with pinned host buffers)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2104_05829_b200 as nk
m = nk.build_box_mesh((1, 1, 1), (20, 20, 20), 7, deformation=("sine", 0.05))
uh = torch.as_tensor(np.random.default_rng(0).standard_normal(m.n_local)).pin_memory()
wh = torch.empty_like(uh).pin_memory()
for ch in (2, 4, 6, 8, 12):
    for _ in range(3):
        nk.apply_stiffness_local(uh, m, out=wh, nchunks=ch)
    ts = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); nk.apply_stiffness_local(uh, m, out=wh, nchunks=ch); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(json.dumps({"nchunks": ch, "ms_med": round(statistics.median(ts), 4),
                      "gdofs": round(m.E * 343 / statistics.median(ts) / 1e6, 3)}))
