"""FP32-path accuracy vs the FP64 oracle on the C2-like test case (GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import paper_1504_05477_b200 as rk
import rsvd_oracle as o
from test_gpu_parity import _fp32_case
for (n, d, k, q) in ((6000, 1200, 50, 10), (20000, 4000, 50, 10)):
    A32 = _fp32_case(n, d, k, q)
    A64 = A32.astype(np.float64)
    ref = o.factorize(o.DenseOp(A64), k, "bk", q=q, seed=0)
    r = rk.block_krylov(A32, rk.RsvdConfig(k=k, variant="bk", q=q, seed=0))
    rel = np.abs(r.approx_singular_values - ref.sigma) / ref.sigma
    cap = o.captured_variance(A64, r.Z.data); cap_ref = o.captured_variance(A64, ref.Z)
    z = r.Z.data
    print(f"{n}x{d}: sigma rel max {rel.max():.2e} median {np.median(rel):.2e}; captured var rel max "
          f"{np.max(np.abs(cap - cap_ref) / cap_ref):.2e}; ZtZ-I {np.max(np.abs(z.T @ z - np.eye(k))):.1e}")
