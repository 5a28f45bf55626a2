"""Ozaki int8 products at the C2 shapes (A 50000 x 10000 FP32): NN width p,
TN width p, for ncu captures (-k k_oz_gemm). GPU only; not a bench number."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops
n, d = 50000, 10000
p = int(sys.argv[1]) if len(sys.argv) > 1 else 50
which = sys.argv[2] if len(sys.argv) > 2 else "both"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
A = torch.randn((n, d), device="cuda")
P = ops.OzPlanes(A)
X = torch.randn((d, p), device="cuda", dtype=torch.float64)
Y = torch.randn((n, p), device="cuda", dtype=torch.float64)
C = torch.empty((n, p), device="cuda", dtype=torch.float64)
W = torch.empty((d, p), device="cuda", dtype=torch.float64)
for name, fn in (("nn", lambda: ops.oz_gemm(P, X, C, 0)), ("tn", lambda: ops.oz_gemm(P, Y, W, 1))):
    if which not in ("both", name):
        continue
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name} p={p}: {ms:.3f} ms, {6 * n * d / ms / 1e6:.0f} GB/s of A planes, "
          f"{27 * 2 * n * d * 64 * (p + 63) // 64 / ms / 1e9:.0f} int8 TOPS (27 planes pairs)", flush=True)
