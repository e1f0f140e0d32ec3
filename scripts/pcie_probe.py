"""Host<->device link probe: pinned H2D, D2H and concurrent H2D+D2H of the
BK5 field size (32.8 MB) -- the ceiling for the e2e path."""
import json, torch
n = 4096000
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def both():
    m = torch.cuda.current_stream()
    s1.wait_stream(m); s2.wait_stream(m)
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    m.wait_stream(s1); m.wait_stream(s2)
h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
bo = t(both)
B = 8 * n
print(json.dumps({"bytes": B, "h2d_GBs": round(B / h2d / 1e6, 1), "d2h_GBs": round(B / d2h / 1e6, 1),
                  "both_ms": round(bo, 4), "both_GBs_total": round(2 * B / bo / 1e6, 1),
                  "e2e_floor_ms": round(bo, 4)}))
