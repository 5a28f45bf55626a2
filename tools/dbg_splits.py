import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
from paper_1504_05477_b200.krylov import rows_buffer
m, n, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, k, generator=g, device="cuda")
B = torch.randn(k, n, generator=g, device="cuda")
C = torch.empty(m, n, device="cuda")
ops.gemm_nn(A, B, C, algo=2)
ref = (A.double() @ B.double())
err = (C.double() - ref).abs() / ref.abs().max()
print(os.environ.get("RSVD_TC_SPLITS"), "max err", float(err.max()))
bad = (err > 1e-5).nonzero()
if bad.numel():
    rows = bad[:, 0].unique()
    print("bad rows:", rows.numel(), "first", rows[:10].tolist(), "last", rows[-5:].tolist(), "cols", bad[:, 1].unique()[:10].tolist())
