"""Build a variant of librsvd_b200.so with extra -D flags on gemm_tc.cu and run
a tool against it. Usage:
  python tools/variant.py build NAME -DFOO -DBAR=1
  python tools/variant.py run NAME tools/some_tool.py args..."""
import glob, os, runpy, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if sys.argv[1] == "build":
    from paper_1504_05477_b200 import build as B
    name, defs = sys.argv[2], sys.argv[3:]
    src = os.path.join(B.CSRC, "gemm_tc.cu")
    if defs and defs[0].endswith(".cu"):  # alternative gemm_tc.cu source (must sit in csrc/ for its includes)
        src = defs.pop(0)
    B.build()
    objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if not o.endswith("gemm_tc.cu.o")]
    os.makedirs(os.path.join(ROOT, "tools", "vbin"), exist_ok=True)
    obj = os.path.join(ROOT, "tools", "vbin", f"gemm_tc_{name}.o")
    subprocess.check_call([B.NVCC] + B.NVCC_FLAGS + ["-I", B.CSRC] + defs + ["-c", src, "-o", obj])
    lib = os.path.join(ROOT, "tools", "vbin", f"librsvd_{name}.so")
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib, obj] + objs + ["-lcudart", "-lcuda"])
    print("built", lib)
else:
    from paper_1504_05477_b200 import _lib
    _lib.LIB_PATH = os.path.join(ROOT, "tools", "vbin", f"librsvd_{sys.argv[2]}.so")
    sys.argv = sys.argv[3:]
    runpy.run_path(sys.argv[0], run_name="__main__")
