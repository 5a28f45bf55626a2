import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops
from paper_1504_05477_b200.krylov import rows_buffer
n, p = 50000, 50
g = torch.Generator(device="cuda").manual_seed(0)
X = rows_buffer(n, p, torch.float32, "cuda"); X.copy_(torch.randn(n, p, generator=g, device="cuda"))
Y = rows_buffer(n, p, torch.float32, "cuda")
T = torch.randn(p, p, generator=g, device="cuda")
G = torch.empty(p, p, dtype=torch.float64, device="cuda")
for _ in range(3):
    ops.gemm_nn(X, T, Y, algo=4)
    ops.gram(X, G, algo=4)
torch.cuda.synchronize()
print("ok")
