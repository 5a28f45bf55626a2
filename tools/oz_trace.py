"""Per-CTA phase stamps (globaltimer) of the digit-plane GEMM: run under
tools/variant.py with a -DRSVD_OZ_TRACE build. Args: jp (basis NN at the C2
shape, 0 = chain NN)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1504_05477_b200 import device as ops, _lib
jp = int(sys.argv[1]) if len(sys.argv) > 1 else 50
n, w, p = 50000, 600, 50
if jp > 0:
    Q = torch.randn((n, w), device="cuda", dtype=torch.float64) / n ** 0.5
    B = ops.OzBasis(n, w, Q.device)
    for c0 in range(0, w, p):
        B.slice(Q, c0, p)
    V = torch.randn((n, p), device="cuda", dtype=torch.float64)
    C = torch.randn((jp, p), device="cuda", dtype=torch.float64)
    fn = lambda: B.gemm(0, jp, C, V, alpha=-1.0, beta=1.0)  # noqa: E731
else:
    A = torch.randn((n, 10000), device="cuda")
    P = ops.OzPlanes(A)
    X = torch.randn((10000, p), device="cuda", dtype=torch.float64)
    Y = torch.empty((n, p), device="cuda", dtype=torch.float64)
    fn = lambda: ops.oz_gemm(P, X, Y, 0)  # noqa: E731
fn(); torch.cuda.synchronize(); fn(); torch.cuda.synchronize()
L = _lib.load()
L.rsvd_debug_oz_trace.argtypes = [ctypes.c_void_p]
buf = np.zeros((512, 5), dtype=np.uint64)
L.rsvd_debug_oz_trace(ctypes.c_void_p(buf.ctypes.data))
t0 = buf[buf[:, 0] > 0, 0].min()
ok = buf[:, 0] > 0
T = (buf[ok].astype(np.int64) - int(t0)) / 1e3  # us
print("CTAs", ok.sum())
print("setup (start->after sync) us: median %.2f max %.2f" % (np.median(T[:, 1] - T[:, 0]), np.max(T[:, 1] - T[:, 0])))
print("mainloop (sync->acc_full) us: median %.2f" % np.median(T[:, 2] - T[:, 1]))
print("epilogue (acc_full->done) us: median %.2f" % np.median(T[:, 3] - T[:, 2]))
print("teardown us: median %.2f" % np.median(T[:, 4] - T[:, 3]))
order = np.argsort(T[:, 0])
for i in order[:: max(1, len(order) // 12)]:
    print(" start %.1f setup %.2f main %.2f epi %.2f end %.1f" % (T[i, 0], T[i, 1] - T[i, 0], T[i, 2] - T[i, 1], T[i, 3] - T[i, 2], T[i, 4]))
