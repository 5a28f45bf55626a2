"""One chain-shaped and one projection-shaped 3xTF32 NN product, eager, for an
ncu stall/instruction-fetch look. Debug tool."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
from paper_1504_05477_b200.krylov import rows_buffer
g = torch.Generator(device="cuda").manual_seed(0)
n, p = 50000, 50
for K in (10000, 550):
    A = rows_buffer(n, K, torch.float32, "cuda"); A.copy_(torch.randn(n, K, generator=g, device="cuda"))
    B = torch.randn(K, p, generator=g, device="cuda")
    C = rows_buffer(n, p, torch.float32, "cuda")
    for _ in range(2):
        ops.gemm_nn(A, B, C, algo=2)
    torch.cuda.synchronize()
    del A
