"""Time the FP64 (reference-faithful) path on C2's FP32 A upcast to FP64, the
way the reference itself computes on FP32 input (matrix.py:80). GPU only."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1504_05477_b200 import rsvd, matrix as mx
from paper_1504_05477_b200.operators import DenseDeviceOp

cfgd = bench.CONFIGS["c2"]
cfg = rsvd.RsvdConfig(k=cfgd["k"], variant=cfgd["variant"], q=cfgd["q"], seed=0)
A64 = bench.make_matrix(cfgd, "cuda").double()
op = DenseDeviceOp(A64)
Pi = mx.gaussian(cfgd["d"], cfg.p, mx.SeededRng(0)).data
for mode in ("eager", "graph"):
    g = rsvd.GraphedFactorization(op, cfg) if mode == "graph" else None
    run = (lambda: g.run(Pi)) if g else (lambda: rsvd.run_device(op, cfg, Pi=Pi))
    run(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        df = run()
    torch.cuda.synchronize()
    print(f"C2 fp64 {mode}: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms", flush=True)
# per-kernel breakdown
from torch.profiler import profile, ProfilerActivity
import collections
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rsvd.run_device(op, cfg, Pi=Pi); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        agg[ev.name[:70]][0] += ev.device_time_total / 1e3
        agg[ev.name[:70]][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"total kernel time {tot:.1f} ms")
for k_, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:12]:
    print(f"  {t:8.2f} ms {c:5d}  {k_}")
