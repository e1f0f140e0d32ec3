import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2104_05829_b200 as nk
m = nk.build_box_mesh((1, 1, 1), (14, 14, 14), 12, deformation=("sine", 0.05))
u = torch.randn(m.n_local, dtype=torch.float64, device="cuda")
w = torch.empty_like(u)
for _ in range(3):
    nk.apply_stiffness_local(u, m, out=w)
torch.cuda.synchronize()
