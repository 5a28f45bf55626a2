import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
p = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(0)
v = rng.standard_normal((2000, p))
G = torch.from_numpy(v.T @ v).cuda()
T = torch.empty((p, p), dtype=torch.float64, device="cuda")
mask = torch.empty(p, dtype=torch.int32, device="cuda")
ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
for _ in range(5):
    ops.chol_deflate(G, None, 1e-14, T, mask, ndef)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ops.chol_deflate(G, None, 1e-14, T, mask, ndef)
e1.record(); torch.cuda.synchronize()
print(f"chol_deflate p={p}: {e0.elapsed_time(e1)/20*1e3:.1f} us")
