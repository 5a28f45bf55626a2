import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
p = int(sys.argv[1])
rng = np.random.default_rng(0)
v = rng.standard_normal((2000, p))
G = torch.from_numpy(v.T @ v).cuda()
T = torch.empty((p, p), dtype=torch.float64, device="cuda")
mask = torch.empty(p, dtype=torch.int32, device="cuda")
ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
for _ in range(3):
    ops.chol_deflate(G, None, 1e-14, T, mask, ndef)
torch.cuda.synchronize(); print("ok")
