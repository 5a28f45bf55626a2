"""Standalone timing of the FP64 skinny products of the orthonormalization at
C2's block shape: V T (50000 x 50 x 50, gemm_nn) and the Gram V^T V (gemm_tn +
ordered reduce). RSVD_DNN_RING=1 / RSVD_DTN_BK16=1 select the previous
configurations. GPU only; not a bench number."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1504_05477_b200 import device as ops

n, p = 50000, 50
K = torch.randn((n, 600), device="cuda", dtype=torch.float64)
V = K[:, 100:150]
T = torch.randn((p, p), device="cuda", dtype=torch.float64)
out = torch.empty((n, 52), device="cuda", dtype=torch.float64)[:, :p]
G = torch.empty((p, p), device="cuda", dtype=torch.float64)


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print(f"V T -> out: {timed(lambda: ops.gemm_nn(V, T, out)):.1f} us; "
      f"out += V T: {timed(lambda: ops.gemm_nn(V, T, out, alpha=-1.0, beta=1.0)):.1f} us; "
      f"Gram: {timed(lambda: ops.gram(V, G)):.1f} us; "
      f"chol p=50: {timed(lambda: ops.chol_deflate(G @ G.T + 50 * torch.eye(p, device='cuda', dtype=torch.float64), None, 1e-14, T.clone(), torch.empty(p, dtype=torch.int32, device='cuda'), torch.zeros(2, dtype=torch.int32, device='cuda'))):.1f} us (with torch setup)")

# floor for these shapes: a strided copy of the same block (read 20 MB, write 20 MB)
print(f"torch copy V -> out: {timed(lambda: out.copy_(V)):.1f} us; convert kernel: {timed(lambda: ops.convert(V, out)):.1f} us; "
      f"colreduce: {timed(lambda: ops.colreduce(V, True)):.1f} us")
Vc = torch.randn((n, p), device="cuda", dtype=torch.float64)
oc = torch.empty((n, p), device="cuda", dtype=torch.float64)
print(f"contiguous operands: V T {timed(lambda: ops.gemm_nn(Vc, T, oc)):.1f} us, Gram {timed(lambda: ops.gram(Vc, G)):.1f} us, "
      f"copy {timed(lambda: oc.copy_(Vc)):.1f} us")
