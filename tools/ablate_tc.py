"""Build ablation variants of the tcgen05 GEMM (RSVD_TC_ABLATE bits, see
gemm_tc.cu) as tools/bin/librsvd_abl<N>.so and time the C2 chain products
with each. Usage: python tools/ablate_tc.py build 1 2 4 8 ; python tools/ablate_tc.py run 0 1 2 ..."""
import glob, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1504_05477_b200 import build as B

def build(v):
    B.build()
    objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if not o.endswith("gemm_tc.cu.o")]
    os.makedirs(os.path.join(ROOT, "tools", "bin"), exist_ok=True)
    obj = os.path.join(ROOT, "tools", "bin", f"gemm_tc_abl{v}.o")
    subprocess.check_call([B.NVCC] + B.NVCC_FLAGS + [f"-DRSVD_TC_ABLATE={v}", "-c",
                           os.path.join(B.CSRC, "gemm_tc.cu"), "-o", obj])
    lib = os.path.join(ROOT, "tools", "bin", f"librsvd_abl{v}.so")
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib, obj] + objs + ["-lcudart", "-lcuda"])
    print("built", lib)

def run(v):
    from paper_1504_05477_b200 import _lib
    if v != "0":
        _lib.LIB_PATH = os.path.join(ROOT, "tools", "bin", f"librsvd_abl{v}.so")
    import runpy
    print(f"ablate {v}: ", end="", flush=True)
    runpy.run_path(os.path.join(ROOT, "tools", "prof_products.py"))

if __name__ == "__main__":
    if sys.argv[1] == "build":
        for v in sys.argv[2:]:
            build(v)
    else:
        run(sys.argv[2])
