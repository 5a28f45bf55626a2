import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
m, k, n = 50000, 10112, 50
S = int(os.environ.get("RSVD_TC_SPLITS", "9"))
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, k, generator=g, device="cuda")
B = torch.randn(m, n, generator=g, device="cuda")
C = torch.empty(k, n, device="cuda", dtype=torch.float64)
ops.gemm_tn(A, B, C, algo=2)
torch.cuda.synchronize()
ws = ops.WS.buf[0][: S * k * n * 4].view(torch.float32).view(S, k, n).double()
kps = -(-(-(-m // S)) // 32) * 32
bad = []
for s in range(S):
    r0, r1 = s * kps, min(m, (s + 1) * kps)
    P = A[r0:r1].double().T @ B[r0:r1].double()
    e = ((ws[s] - P).abs().view(-1, 128, n).amax(dim=(1, 2)) / P.abs().max()).cpu().numpy()
    for t in np.nonzero(e > 1e-5)[0]:
        u = t * S + s
        bad.append((s, int(t), u, u % 148, u // 148))
print("S", S, "bad (split, tile, unit, cta, round):", bad[:25], "total", len(bad))
