"""Per-k-block pipeline trace of the tcgen05 chain GEMM (A.X at C2 shape).
`python tools/trace_tc.py build` compiles gemm_tc.cu with -DRSVD_TC_TRACE into
tools/bin/librsvd_trace.so; `python tools/trace_tc.py run` (GPU) runs one A.X
and prints, per traced CTA, medians of the stage-to-stage intervals (cycles).
Series: 0 A-TMA issue, 1 conv sees A, 2 conv got TMEM stage, 3 conv done,
4 MMA wants stage, 5 MMA sees conv, 6 MMA sees B, 7 MMA committed."""
import ctypes, glob, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "tools", "bin", "librsvd_trace.so")

def build(extra=()):
    from paper_1504_05477_b200 import build as B
    B.build()
    objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if not o.endswith("gemm_tc.cu.o")]
    obj = os.path.join(ROOT, "tools", "bin", "gemm_tc_trace.o")
    subprocess.check_call([B.NVCC] + B.NVCC_FLAGS + ["-DRSVD_TC_TRACE"] + list(extra) + ["-c", os.path.join(B.CSRC, "gemm_tc.cu"), "-o", obj])
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", LIB, obj] + objs + ["-lcudart", "-lcuda"])
    print("built", LIB)

def run():
    from paper_1504_05477_b200 import _lib
    print("trace lib", LIB)
    _lib.LIB_PATH = LIB
    import torch
    from paper_1504_05477_b200.operators import DenseDeviceOp
    n, d, p = 50000, 10000, 50
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((n, d), generator=g, device="cuda") / 100.0
    op = DenseDeviceOp(A)
    X = torch.randn((d, p), generator=g, device="cuda")
    Y = torch.empty((n, p), device="cuda")
    for _ in range(3):
        op.apply(X, Y)
    torch.cuda.synchronize()
    L = _lib.load()
    buf = np.zeros((2, 8, 512), dtype=np.int64)
    L.rsvd_debug_tc_trace.argtypes = [ctypes.c_void_p]
    assert L.rsvd_debug_tc_trace(buf.ctypes.data) == 0
    nkb = 313
    for c, name in ((0, "CTA 0"), (1, "CTA 200")):
        t = buf[c, :, :nkb].astype(np.float64)
        mk = buf[c, :4, 511].astype(np.float64)
        base = mk[0]
        print(f"{name}: setup {mk[1]-base:.0f}, first A issue {buf[c,0,0]-base:.0f}, last MMA commit {buf[c,7,nkb-1]-base:.0f}, last drain {mk[2]-base:.0f}, epilogue done {mk[3]-base:.0f}")
        t -= t[0, 0]
        med = lambda x: float(np.median(x[20:-20]))
        print(f"{name}: total {t[7, -1] - t[0, 0]:.0f} cyc for {nkb} k-blocks = {(t[7, -1] - t[0, 0]) / nkb:.0f} cyc/kb")
        print(f"  A-TMA issue period       {med(np.diff(t[0])):7.0f}")
        print(f"  TMA latency (0->1)       {med(t[1] - t[0]):7.0f}")
        print(f"  conv waits TMEM (1->2)   {med(t[2] - t[1]):7.0f}")
        print(f"  conv work (2->3)         {med(t[3] - t[2]):7.0f}")
        print(f"  MMA waits (4->6)         {med(t[6] - t[4]):7.0f}")
        print(f"  MMA issue (6->7)         {med(t[7] - t[6]):7.0f}")
        print(f"  MMA commit period        {med(np.diff(t[7])):7.0f}")
        print(f"  A-TMA issue lag vs MMA commit of kb-8 (0[kb]-7[kb-8]) {med(t[0, 8:] - t[7, :-8]):7.0f}")
        print(f"  TMEM stage turnaround (2[kb]-7[kb-ST]) ST=4: {med(t[2, 4:] - t[7, :-4]):7.0f}")
        for kb in (30, 31, 32, 33, 150, 151):
            print("   kb", kb, " ".join(f"{v:9.0f}" for v in t[:, kb]))

if __name__ == "__main__":
    if sys.argv[1] == "build":
        if len(sys.argv) > 2:
            LIB = LIB.replace(".so", f"_{sys.argv[2]}.so")
        build([f"-DRSVD_TC_ABLATE={sys.argv[2]}"] if len(sys.argv) > 2 else [])
    else:
        if len(sys.argv) > 2:
            LIB = LIB.replace(".so", f"_{sys.argv[2]}.so")
        run()
