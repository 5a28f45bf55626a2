import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
w, k = 600, 50
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(w, w, generator=g, device="cuda", dtype=torch.float64)
M = X @ X.T
for _ in range(2):
    ops.syev_topk(M, k)
torch.cuda.synchronize(); print("ok")
