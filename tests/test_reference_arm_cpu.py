"""bench.py's reference arm on the host: it must run the oracle port on a
host-generated A without importing anything from the product package (and
without CUDA), and its input generator must produce the configured spectrum."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_host_generator_spectrum():
    cfgd = dict(n=3000, d=400, spectrum="pow", noise=0.0)
    A = bench.make_matrix_host(cfgd, seed=5)
    assert A.dtype == np.float32 and A.shape == (3000, 400)
    s = np.linalg.svd(A.astype(np.float64), compute_uv=False)
    ref = np.arange(1, 401, dtype=np.float64) ** -0.5
    assert np.max(np.abs(s - ref) / ref) < 1e-5  # FP32 rounding of A only
    # deterministic
    assert np.array_equal(A, bench.make_matrix_host(cfgd, seed=5))


def test_reference_arm_imports_no_product_code():
    code = f"""
import sys, json
sys.path.insert(0, {ROOT!r})
import bench
bench.CONFIGS["tiny"] = dict(n=1500, d=300, k=10, q=4, spectrum="pow", noise=1e-3, variant="bk", mode="exact")
sys.argv = ["bench.py", "--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "1"]
bench.main()
bad = [m for m in sys.modules if m.startswith("paper_1504_05477_b200")]
print(json.dumps({{"product_modules": bad, "cuda_init": bool(sys.modules.get("torch") and
                  sys.modules["torch"].cuda.is_initialized())}}))
"""
    env = dict(os.environ, OPENBLAS_NUM_THREADS="2", OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "port"
    assert line["config"]["q_eff"] == 5 and line["config"]["krylov_width"] == 60
    assert probe["product_modules"] == [] and not probe["cuda_init"]
