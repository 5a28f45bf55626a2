"""FP64 DMMA products at the C2 orthonormalization shapes (n = 50000, p = 50,
prefix jp = 550): Q_p^T V (TN) and Q_p C (NN), for ncu. GPU only."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops
n, p = 50000, 50
jp = int(sys.argv[1]) if len(sys.argv) > 1 else 550
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
Q = torch.randn((n, jp), device="cuda", dtype=torch.float64)
V = torch.randn((n, p), device="cuda", dtype=torch.float64)
C = torch.empty((jp, p), device="cuda", dtype=torch.float64)
for name, fn in (("tn", lambda: ops.gemm_tn(Q, V, C)), ("nn", lambda: ops.gemm_nn(Q, C, V, alpha=-1.0, beta=1.0)),
                 ("gram", lambda: ops.gram(V))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * n * (jp if name != "gram" else p) * p
    print(f"{name} jp={jp}: {ms*1e3:.1f} us, {fl/ms/1e9:.1f} TFLOP/s", flush=True)
