import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
m, n, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, k, generator=g, device="cuda")
B = torch.randn(k, n, generator=g, device="cuda")
C = torch.empty(m, n, device="cuda")
ops.gemm_nn(A, B, C, algo=2)
ref = (A.double() @ B.double())
err = ((C.double() - ref).abs() / ref.abs().max()).view(-1, 128, n).amax(dim=(1, 2)).cpu().numpy()
bad = np.nonzero(err > 1e-5)[0]
print(os.environ.get("RSVD_TC_SPLITS"), m, n, k, "bad tiles", len(bad), bad[:12].tolist(), "max", err.max())
