"""Per-phase clock64 trace of k_chol_blk (debug build with -DRSVD_CHOL_TRACE).
`build` makes tools/bin/librsvd_ctrace.so; `run P...` prints phase cycles."""
import ctypes, glob, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "tools", "bin", "librsvd_ctrace.so")
if sys.argv[1] == "build":
    from paper_1504_05477_b200 import build as B
    B.build()
    objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if not o.endswith("small_dense.cu.o")]
    obj = os.path.join(ROOT, "tools", "bin", "small_dense_trace.o")
    subprocess.check_call([B.NVCC] + B.NVCC_FLAGS + ["-DRSVD_CHOL_TRACE", "-c", os.path.join(B.CSRC, "small_dense.cu"), "-o", obj])
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", LIB, obj] + objs + ["-lcudart", "-lcuda"])
    print("built", LIB)
    sys.exit()
from paper_1504_05477_b200 import _lib
_lib.LIB_PATH = LIB
import torch
from paper_1504_05477_b200 import device as ops
L = _lib.load()
L.rsvd_debug_chol_trace.argtypes = [ctypes.c_void_p]
for p in [int(x) for x in sys.argv[2:]]:
    rng = np.random.default_rng(0)
    v = rng.standard_normal((2000, p))
    G = torch.from_numpy(v.T @ v).cuda()
    T = torch.empty((p, p), dtype=torch.float64, device="cuda")
    mask = torch.empty(p, dtype=torch.int32, device="cuda")
    ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
    for _ in range(3):
        ops.chol_deflate(G, None, 1e-14, T, mask, ndef)
    torch.cuda.synchronize()
    buf = np.zeros(64, dtype=np.int64)
    L.rsvd_debug_chol_trace(buf.ctypes.data)
    print(f"p={p}: factor {buf[1] - buf[0]} cycles, invert {buf[2] - buf[1]}, output {buf[3] - buf[2]}; "
          f"k_chol_blk phases: diag warp {buf[8]}, panel columns {buf[9]}, trailing update {buf[10]}, "
          f"inverse columns {buf[11]}, inverse pass {buf[12]}")
