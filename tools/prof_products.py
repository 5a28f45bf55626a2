"""The C2 Krylov-chain products alone (A.X and A^T.Y at width p = 50, FP32
A 50000 x 10000), for ncu captures of the dominant kernel."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200.operators import DenseDeviceOp
n, d, p = 50000, 10000, 50
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((n, d), generator=g, device="cuda") / 100.0
op = DenseDeviceOp(A)
X = torch.randn((d, p), generator=g, device="cuda")
Y = torch.empty((n, p), device="cuda")
C = torch.empty((d, p), device="cuda")
for _ in range(3):
    op.apply(X, Y)
    op.apply_t(Y, C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    op.apply(X, Y)
e1.record(); torch.cuda.synchronize()
ax = e0.elapsed_time(e1) / 10
e0.record()
for _ in range(10):
    op.apply_t(Y, C)
e1.record(); torch.cuda.synchronize()
aty = e0.elapsed_time(e1) / 10
byt = n * d * 4 + (n + d) * p * 4
print(f"A.X {ax:.3f} ms {byt/ax/1e6:.0f} GB/s ; A^T.Y {aty:.3f} ms {byt/aty/1e6:.0f} GB/s")
