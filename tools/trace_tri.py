"""clock64 trace of k_tridiag_cluster columns (debug build -DRSVD_TRI_TRACE)."""
import ctypes, glob, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "tools", "bin", "librsvd_tritrace.so")
if sys.argv[1] == "build":
    from paper_1504_05477_b200 import build as B
    B.build()
    objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if not o.endswith("syev.cu.o")]
    obj = os.path.join(ROOT, "tools", "bin", "syev_trace.o")
    subprocess.check_call([B.NVCC] + B.NVCC_FLAGS + ["-DRSVD_TRI_TRACE", "-c", os.path.join(B.CSRC, "syev.cu"), "-o", obj])
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", LIB, obj] + objs + ["-lcudart", "-lcuda"])
    print("built"); sys.exit()
from paper_1504_05477_b200 import _lib
_lib.LIB_PATH = LIB
import torch
from paper_1504_05477_b200 import device as ops
w, k = 600, 50
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(w, w, generator=g, device="cuda", dtype=torch.float64)
M = X @ X.T
for _ in range(2):
    ev, evec, info = ops.syev_topk(M, k) if hasattr(ops, "syev_topk") else (None, None, None)
torch.cuda.synchronize()
L = _lib.load(); L.rsvd_debug_tri_trace.argtypes = [ctypes.c_void_p]
buf = np.zeros((64, 8), dtype=np.int64); L.rsvd_debug_tri_trace(buf.ctypes.data)
d = np.diff(buf[8:40, :7], axis=1)
names = ["owner HH", "sync1", "u fetch+matvec", "sync2", "gather p + q", "rank-2 update"]
per = np.median(d, axis=0)
print("median cycles per column phase:", dict(zip(names, per.astype(int))), "total", int(np.median(buf[9:40, 0] - buf[8:39, 0])))
