"""Per-tile error map of the tcgen05 GEMM (rows whose error exceeds 1e-5, grouped
by 128-row tile): the check that caught the converters' A-stage release race. GPU only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops
from paper_1504_05477_b200._lib import GEMM_TC_3XTF32 as TC

for (m, n, k) in [(20000, 128, 600), (20000, 128, 640), (20000, 96, 600), (20000, 64, 600), (40000, 128, 4096),
                  (20000, 200, 600)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn((m, k), generator=g, device="cuda")
    B = torch.randn((k, n), generator=g, device="cuda")
    C = torch.empty((m, n), device="cuda")
    ops.gemm_nn(A, B, C, algo=TC)
    ref = A.double() @ B.double()
    err = (C.double() - ref).abs().amax(1) / ref.abs().max()
    bad = torch.nonzero(err > 1e-5).flatten()
    tiles = sorted(set((bad // 128).tolist()))
    print(f"NN {m}x{n}x{k}: max {err.max().item():.2e}, bad rows {bad.numel()}, bad tiles {tiles[:20]}", flush=True)
    Y = torch.randn((m, n), generator=g, device="cuda")
    Ct = torch.empty((k, n), device="cuda")
    ops.gemm_tn(A, Y, Ct, algo=TC)
    ref = A.double().T @ Y.double()
    e = ((Ct.double() - ref).abs().max() / ref.abs().max()).item()
    print(f"TN {m}x{n}x{k}: max {e:.2e}", flush=True)
