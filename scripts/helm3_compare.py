"""3-component Helmholtz apply: batched pencil3 (G read once) vs three scalar
BK5 launches (G read three times), L2 flushed before each timed apply."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05829_b200 as nk
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
for N, ne in ((7, 20), (9, 16), (9, 24), (5, 29)):
    m = nk.build_box_mesh((1, 1, 1), (ne, ne, ne), N, deformation=("sine", 0.05))
    n = m.n_local
    u3 = torch.randn(3 * n, dtype=torch.float64, device="cuda")
    w3 = torch.empty_like(u3)

    def batched():
        nk.apply_helmholtz_local(u3, m, 1e-3, 1833.0, ncomp=3, out=w3)

    def scalar():
        for c in range(3):
            nk.apply_helmholtz_local(u3[c * n:(c + 1) * n], m, 1e-3, 1833.0, ncomp=1,
                                     out=w3[c * n:(c + 1) * n])

    res = {"N": N, "E": m.E}
    for name, fn in (("batched_ms", batched), ("scalar3_ms", scalar)):
        ts = []
        for rep in range(15):
            flush.fill_(rep)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); b.synchronize()
            if rep >= 3:
                ts.append(a.elapsed_time(b))
        res[name] = round(statistics.median(ts), 4)
    res["batched_over_scalar"] = round(res["batched_ms"] / res["scalar3_ms"], 3)
    print(json.dumps(res), flush=True)
