import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
m, n, k = 18944, 50, 2048
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, k, generator=g, device="cuda").double()
B = torch.randn(k, n, generator=g, device="cuda").double()
C = torch.empty(m, n, device="cuda")
ops.gemm_nn(A.float(), B.float(), C, algo=2)
C = C.double()
P = [A[:, :1024] @ B[:1024], A[:, 1024:] @ B[1024:]]
ref = P[0] + P[1]
t = lambda X, i: X[i * 128:(i + 1) * 128]
for T in (74, 75, 80, 100):
    d = t(C, T) - t(ref, T)
    c = 2 * (T - 74)  # CTA of (tile T, split 0); split 1 is CTA c+1
    prev0, prev1 = t(P[0], c // 2), t(P[1], (c + 1) // 2)
    err = float(d.abs().max())
    for name, cand in (("prev split0 tile", prev0), ("prev split1 tile", prev1), ("both", prev0 + prev1)):
        r = float((d - cand).abs().max())
        print(f"tile {T}: |C-ref| {err:.3e}  |C-ref-{name}| {r:.3e}")
    rows_bad = (d.abs().amax(dim=1) > 1e-3).nonzero().flatten().tolist()
    print("   bad rows", rows_bad[:40])
