"""C5 chain-product shapes (A 500000 x 2000 FP32, width 200) through the
3xTF32 tcgen05 kernels, with and without the centering epilogue, against
the C4 shape (1e6 x 4096). TFLOP/s vs measured TF32/3. GPU only."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
which = sys.argv[2] if len(sys.argv) > 2 else "all"
res = {}
for label, n, d in (("c5", 500000, 2000), ("c4", 1000000, 4096)):
    if which not in ("all", label):
        continue
    b = 200
    A = torch.randn((n, d), device="cuda")
    X = torch.randn((d, b), device="cuda")
    Y = torch.randn((n, b), device="cuda")
    Yo = torch.empty((n, b), device="cuda")
    Xo = torch.empty((d, b), device="cuda")
    mu = torch.randn(d, device="cuda", dtype=torch.float64)
    rs = torch.randn((1, b), device="cuda", dtype=torch.float64)
    cs = torch.randn(b, device="cuda", dtype=torch.float64)
    fl = 2.0 * n * d * b
    for name, fn in (("A.X", lambda: ops.gemm_nn(A, X, Yo)), ("A^T.Y", lambda: ops.gemm_tn(A, Y, Xo)),
                     ("A.X centered", lambda: ops.gemm_nn(A, X, Yo, row_sub=rs)),
                     ("A^T.Y centered", lambda: ops.gemm_tn(A, Y, Xo, mu=mu, colsum_b=cs))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[f"{label} {name}"] = {"ms": ms, "tflops": fl / ms / 1e9, "frac_tf32_3": fl / ms / 1e9 / (755.8 / 3)}
    del A, X, Y, Yo, Xo
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
