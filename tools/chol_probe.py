"""p = 50 Cholesky-with-deflation (the orthonormalization's small step):
time per call, for ncu. GPU only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops, krylov
p = int(sys.argv[1]) if len(sys.argv) > 1 else 50
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
V = torch.randn((50000, p), device="cuda", dtype=torch.float64)
G = ops.gram(V)
ws = krylov.Workspace("cuda", p)
f = lambda: ops.chol_deflate(G, None, 1e-14, ws.T, ws.mask, ws.ndef)  # noqa: E731
f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    f()
e1.record(); torch.cuda.synchronize()
print(f"chol p={p}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/call", flush=True)
