"""Build a variant of librsvd_b200.so with extra -D flags on one csrc file
(default gemm_tc.cu) and run a tool against it. Usage:
  python tools/variant.py build NAME [--file sparse.cu | path/alt.cu] -DFOO -DBAR=1
  python tools/variant.py run NAME tools/some_tool.py args..."""
import glob, os, runpy, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VBIN = os.path.join(ROOT, "tools", "vbin")

if sys.argv[1] == "build":
    from paper_1504_05477_b200 import build as B
    name, defs = sys.argv[2], sys.argv[3:]
    fname, src = "gemm_tc.cu", None
    if defs and defs[0] == "--file":
        fname = defs[1]
        defs = defs[2:]
    elif defs and defs[0].endswith(".cu"):  # alternative gemm_tc.cu source
        src = defs.pop(0)
    src = src or os.path.join(B.CSRC, fname)
    B.build()
    objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if not o.endswith(fname + ".o")]
    os.makedirs(VBIN, exist_ok=True)
    obj = os.path.join(VBIN, f"{fname}_{name}.o")
    subprocess.check_call([B.NVCC] + B.NVCC_FLAGS + ["-I", B.CSRC] + defs + ["-c", src, "-o", obj])
    lib = os.path.join(VBIN, f"librsvd_{name}.so")
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib, obj] + objs + ["-lcudart", "-lcuda", "-ldl"])
    print("built", lib)
else:
    from paper_1504_05477_b200 import _lib
    _lib.LIB_PATH = os.path.join(VBIN, f"librsvd_{sys.argv[2]}.so")
    sys.argv = sys.argv[3:]
    runpy.run_path(sys.argv[0], run_name="__main__")
