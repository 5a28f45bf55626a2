"""Per-shape device time of the GEMM-like calls of one factorization
(CUDA events around every ops.gemm_nn / gemm_tn / spmm call, grouped by
(kind, m, n, k)). Random A of the config's shape (the orthonormalization and
Rayleigh-Ritz shapes do not depend on the values). GPU only.
Usage: shape_prof.py c4"""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1504_05477_b200 import device as ops, rsvd, matrix as mx
from paper_1504_05477_b200.operators import DenseDeviceOp

cfgd = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
cfg = rsvd.RsvdConfig(k=cfgd["k"], variant=cfgd["variant"], q=cfgd["q"], seed=0)
n, d = cfgd["n"], cfgd["d"]
A = torch.randn((n, d), device="cuda") / (n ** 0.5)
op = DenseDeviceOp(A, center=bool(cfgd.get("pca")))
Pi = mx.gaussian(d, cfg.p, mx.SeededRng(0)).data
rsvd.run_device(op, cfg, Pi=Pi)
torch.cuda.synchronize()
rec = []
orig = {}
for name in ("gemm_nn", "gemm_tn", "split_b" if hasattr(ops, "split_b") else None):
    if name is None:
        continue
    f = getattr(ops, name)
    orig[name] = f

    def w(*a, _f=f, _n=name, **k):
        A_, B_ = a[0], a[1]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = _f(*a, **k)
        e1.record()
        rec.append((_n, tuple(A_.shape), tuple(B_.shape), str(A_.dtype)[6:], e0, e1))
        return r
    setattr(ops, name, w)
rsvd.run_device(op, cfg, Pi=Pi)
torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
for nm, sa, sb, dt, e0, e1 in rec:
    t = e0.elapsed_time(e1)
    if nm == "gemm_nn":
        fl = 2.0 * sa[0] * sa[1] * sb[1]
    else:
        fl = 2.0 * sa[0] * sa[1] * sb[1]
    key = (nm, sa, sb, dt)
    agg[key][0] += t
    agg[key][1] += 1
    agg[key][2] += fl
tot = sum(v[0] for v in agg.values())
print(f"total {tot:.1f} ms in {len(rec)} calls")
for key, (t, c, fl) in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{t:8.2f} ms x{c:3d}  {fl / t / 1e9:7.1f} TF/s  {key}")
