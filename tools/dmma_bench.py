"""Time the FP64 products (DMMA vs CUDA-core) at the FP64-mode chain shapes.
Debug tool, not shipped:  python tools/dmma_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as D  # noqa: E402
from paper_1504_05477_b200._lib import GEMM_DMMA, GEMM_SIMT  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


g = torch.Generator(device="cuda").manual_seed(0)
SHAPES = [(50000, 10000, 50), (50000, 10000, 600), (2000, 1000, 20), (500000, 2000, 200), (1000000, 200, 200)]
if len(sys.argv) > 1:  # --shape m,k,n (profiling)
    SHAPES = [tuple(int(v) for v in sys.argv[-1].split(","))]
for (m, k, n) in SHAPES:
    A = torch.randn(m, k, device="cuda", dtype=torch.float64, generator=g)
    X = torch.randn(k, n, device="cuda", dtype=torch.float64, generator=g)
    Y = torch.randn(m, n, device="cuda", dtype=torch.float64, generator=g)
    C = torch.empty(m, n, device="cuda", dtype=torch.float64)
    W = torch.empty(k, n, device="cuda", dtype=torch.float64)
    fl = 2.0 * m * n * k
    out = [f"m={m} k={k} n={n}:"]
    for name, algo in (("dmma", GEMM_DMMA), ("simt", GEMM_SIMT)):
        t_nn = timeit(lambda: D.gemm_nn(A, X, C, algo=algo))
        t_tn = timeit(lambda: D.gemm_tn(A, Y, W, algo=algo))
        out.append(f"{name} NN {t_nn:.3f} ms {fl / t_nn / 1e9:.1f} TF | TN {t_tn:.3f} ms {fl / t_tn / 1e9:.1f} TF;")
    t_ref = timeit(lambda: torch.matmul(A, X, out=C))
    out.append(f"torch NN {t_ref:.3f} ms {fl / t_ref / 1e9:.1f} TF")
    print(" ".join(out), flush=True)
    del A, X, Y, C, W
    torch.cuda.empty_cache()
