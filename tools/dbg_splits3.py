import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
m, n, k = 37888, 50, 2048
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, k, generator=g, device="cuda")
for half in ("second", "first"):
    B = torch.randn(k, n, generator=g, device="cuda")
    if half == "second": B[k // 2:] = 0
    else: B[: k // 2] = 0
    C = torch.empty(m, n, device="cuda")
    ops.gemm_nn(A, B, C, algo=2)
    ref = (A.double() @ B.double())
    e = ((C.double() - ref).abs() / ref.abs().max()).view(-1, 4, 32, n)
    tiles = e.amax(dim=(1, 2, 3)).cpu().numpy()
    bad = np.nonzero(tiles > 1e-5)[0]
    print(f"B {half} half zero: bad tiles {len(bad)} {bad[:8].tolist()}")
    if len(bad):
        t = bad[0]
        print("  quarters max err", e[t].amax(dim=(1, 2)).cpu().numpy(), " rows bad in q0:", int((e[t, 0].amax(dim=1) > 1e-5).sum()))
