"""Small launches of the hand-written kernels for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per process): int8 Ozaki GEMMs
(NN, TN, basis planes), 3xTF32 tcgen05 GEMMs (NN, TN), FP64 DMMA products,
the cluster tridiagonalisation (w <= 608) and the grid one (w > 608), the
blocked Cholesky, and one small exact-mode factorization."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1504_05477_b200 import device as ops, rsvd
from paper_1504_05477_b200.operators import DenseDeviceOp

torch.manual_seed(0)
dev = "cuda"
n, d, p = 700, 300, 50
A = torch.randn((n, d), device=dev)
P = ops.OzPlanes(A)
X = torch.randn((d, p), device=dev, dtype=torch.float64)
Y = torch.randn((n, p), device=dev, dtype=torch.float64)
ops.oz_gemm(P, X, torch.empty((n, p), device=dev, dtype=torch.float64), 0)
ops.oz_gemm(P, Y, torch.empty((d, p), device=dev, dtype=torch.float64), 1)
Q, _ = torch.linalg.qr(torch.randn((n, 150), device=dev, dtype=torch.float64))
B = ops.OzBasis(n, 150, dev)
B.slice(Q.contiguous(), 0, 50)
B.slice(Q.contiguous(), 50, 50)
C = torch.empty((100, p), device=dev, dtype=torch.float64)
B.gemm(1, 100, Y, C)
B.gemm(0, 100, C, Y, alpha=-1.0, beta=1.0)
X32, Y32 = X.float(), Y.float()
ops.gemm_nn(A, X32, torch.empty((n, p), device=dev))
ops.gemm_tn(A, Y32, torch.empty((d, p), device=dev))
A64 = A.double()
ops.gemm_nn(A64, X, torch.empty((n, p), device=dev, dtype=torch.float64))
ops.gemm_tn(A64, Y, torch.empty((d, p), device=dev, dtype=torch.float64))
for w in (200, 640):
    M = torch.randn((w, w), device=dev, dtype=torch.float64)
    M = M @ M.T
    ops.syev_topk(M, 10)
G = torch.randn((200, 200), device=dev, dtype=torch.float64)
G = G @ G.T + 200 * torch.eye(200, device=dev, dtype=torch.float64)
from paper_1504_05477_b200 import krylov
ws = krylov.Workspace(dev, 200)
ops.chol_deflate(G, None, 0.0, ws.T, ws.mask, ws.ndef)
cfg = rsvd.RsvdConfig(k=10, variant="bk", q=3, seed=0)
rsvd.run_device(DenseDeviceOp(A, exact=True), cfg)
torch.cuda.synchronize()
print("sanitize_small: ok")
