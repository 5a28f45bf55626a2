"""Gram of an n x 50 FP32 block through the skinny kernels (C2 orthonormalization shape). Debug tool."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
from paper_1504_05477_b200.krylov import rows_buffer
g = torch.Generator(device="cuda").manual_seed(0)
V = rows_buffer(50000, 50, torch.float32, "cuda"); V.copy_(torch.randn(50000, 50, generator=g, device="cuda"))
G = torch.empty(50, 50, dtype=torch.float64, device="cuda")
for _ in range(3): ops.gram(V, G, algo=4)
torch.cuda.synchronize()
