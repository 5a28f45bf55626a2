"""Per-call shapes and CUDA-event times of the FP64 products inside one eager
C2 exact-mode factorization (which DMMA shapes dominate). GPU only."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1504_05477_b200 import rsvd, matrix as mx, device as ops
from paper_1504_05477_b200.operators import DenseDeviceOp

cfgd = bench.CONFIGS["c2"]
cfg = rsvd.RsvdConfig(k=cfgd["k"], variant=cfgd["variant"], q=cfgd["q"], seed=0)
A = bench.make_matrix(cfgd, "cuda")
op = DenseDeviceOp(A, exact=True)
Pi = mx.gaussian(A.shape[1], cfg.p, mx.SeededRng(0)).data
rsvd.run_device(op, cfg, Pi=Pi); torch.cuda.synchronize()
rec = []
def wrap(name, fn):
    def w(A_, B_, C_, *a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(A_, B_, C_, *a, **k); e1.record()
        rec.append((name, tuple(A_.shape), tuple(B_.shape), k.get("pred") is not None, e0, e1))
        return r
    return w
ops.gemm_tn = wrap("tn", ops.gemm_tn)
ops.gemm_nn = wrap("nn", ops.gemm_nn)
rsvd.run_device(op, cfg, Pi=Pi); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for name, sa, sb, pr, e0, e1 in rec:
    key = (name, sa[0] // 1000 * 1000 if sa[0] > 5000 else sa[0], sa[1], sb[1], pr)
    agg[key][0] += 1
    agg[key][1] += e0.elapsed_time(e1)
tot = sum(v[1] for v in agg.values())
print(f"FP64 products: {len(rec)} calls, {tot:.2f} ms (eager, incl. predicated-off)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{v[1]:8.3f} ms  n={v[0]:3d}  {k[0]} A{k[1]}x{k[2]} B..x{k[3]} pred={k[4]}  {v[1]/v[0]*1e3:.0f} us/call")
