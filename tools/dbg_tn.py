import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
m, k, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, k, generator=g, device="cuda")
B = torch.randn(m, n, generator=g, device="cuda")
C = torch.empty(k, n, device="cuda", dtype=torch.float64)
ops.gemm_tn(A, B, C, algo=2)
ref = A.double().T @ B.double()
e = ((C - ref).abs() / ref.abs().max()).view(-1, 128, n).amax(dim=(1, 2)).cpu().numpy() if k % 128 == 0 else ((C - ref).abs() / ref.abs().max()).amax().cpu().numpy()
print(os.environ.get("RSVD_TC_SPLITS"), "TN", m, k, n, "bad tiles", np.nonzero(np.atleast_1d(e) > 1e-5)[0][:10].tolist(), "max", float(np.max(e)))
