"""Is the cold CSR gather limited by the kernel or by the column pattern?
Times the plan product on synthetic CSR matrices of C3's cold shape (200000
rows, ~54 nonzeros per row, 100000 columns, width 100): uniform random
columns with equal row lengths, uniform columns with C3-like lognormal row
lengths, and C3's own cold part. GPU only; not a bench number."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1504_05477_b200 import device as ops
from paper_1504_05477_b200.operators import CsrDeviceOp


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = torch.device("cuda", 0)
n, d, b = 200000, 100000, 100
g = torch.Generator(device=dev).manual_seed(3)
X = torch.randn((d, b), generator=g, device=dev)
out = torch.empty((n, b), device=dev)


def run(label, indptr, col, val):
    plan = ops.SpmmPlan(indptr)
    ms = timed(lambda: ops.spmm_csr_plan(plan, col, val, X, out))
    nplan = ops.SpmmNnzPlan(indptr)
    ms2 = timed(lambda: ops.spmm_nnz_plan(nplan, col, val, X, out))
    nnz = val.numel()
    print(f"{label}: nnz {nnz}, row plan {ms:.3f} ms ({nnz * b * 4 / ms / 1e6:.0f} GB/s of gathered rows), "
          f"nnz plan {ms2:.3f} ms ({nnz * b * 4 / ms2 / 1e6:.0f} GB/s)", flush=True)


# uniform columns, equal rows
per = 54
col = torch.randint(0, d, (n * per,), generator=g, device=dev, dtype=torch.int32)
indptr = (torch.arange(n + 1, device=dev, dtype=torch.int32) * per)
val = torch.rand(n * per, generator=g, device=dev)
run("uniform columns, 54 per row", indptr, col, val)
# uniform columns, lognormal row lengths (mean 54)
lens = torch.clamp(torch.round(torch.exp(torch.randn(n, generator=g, device=dev) + 3.49)), 1, 3000).to(torch.int64)
ip = torch.zeros(n + 1, dtype=torch.int64, device=dev)
ip[1:] = torch.cumsum(lens, 0)
nnz = int(ip[-1])
col2 = torch.randint(0, d, (nnz,), generator=g, device=dev, dtype=torch.int32)
val2 = torch.rand(nnz, generator=g, device=dev)
run("uniform columns, lognormal rows", ip.to(torch.int32), col2, val2)
# C3's cold part
cfgd = bench.CONFIGS["c3"]
indptr3, col3, val3 = bench.make_csr(cfgd, dev)
op = CsrDeviceOp(indptr3, col3, val3, d)
run("C3 cold CSR (columns beyond the 405-column panel)", op.indptr, op.col, op.val)
# the same nonzeros with their columns shuffled among themselves (same multiset, no row structure)
perm = torch.randperm(op.col.numel(), generator=g, device=dev)
run("C3 cold CSR, columns permuted across rows", op.indptr, op.col[perm].contiguous(), op.val)
