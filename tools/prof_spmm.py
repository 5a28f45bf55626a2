"""C3 SpMM timings: A.X (CSR, width p) and A^T.Y (CSR of A^T), GB/s against
the algorithmic bytes of SURVEY 8(d). GPU only."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import bench
from paper_1504_05477_b200.operators import CsrDeviceOp
cfgd = bench.CONFIGS["c3"]
t0 = time.time()
indptr, col, val = bench.make_csr(cfgd, "cuda")
print(f"C3 generated in {time.time()-t0:.1f}s nnz={val.numel()}")
n, d, p = cfgd["n"], cfgd["d"], cfgd["k"]
t0 = time.time()
op = CsrDeviceOp(indptr, col, val, d)
torch.cuda.synchronize(); print(f"CSR^T built in {time.time()-t0:.2f}s; max row nnz A {int((indptr[1:]-indptr[:-1]).max())}, A^T {int((op.t_indptr[1:]-op.t_indptr[:-1]).max())}")
X = torch.randn(d, p, device="cuda"); Y = torch.empty(n, p, device="cuda"); C = torch.empty(d, p, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps
nnz = val.numel()
for name, fn, rows in (("A.X", lambda: op.apply(X, Y), n), ("A^T.Y", lambda: op.apply_t(Y, C), d)):
    ms = t(fn)
    byt = nnz * 8 + (rows + 1) * 4 + (n + d) * p * 4
    print(f"{name}: {ms:.3f} ms  {byt/ms/1e6:.0f} GB/s algorithmic ({byt/1e6:.0f} MB)")
