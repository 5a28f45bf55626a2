"""Digit-plane projections against an orthonormal basis prefix at the C2
shapes (n = 50000, p = 50, prefix jp): Q_p^T V and V - Q_p C. For ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops
n, w, p = 50000, 600, 50
jp = int(sys.argv[1]) if len(sys.argv) > 1 else 550
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
Q = torch.randn((n, w), device="cuda", dtype=torch.float64) / n ** 0.5
B = ops.OzBasis(n, w, Q.device)
for c0 in range(0, w, p):
    B.slice(Q, c0, p)
V = torch.randn((n, p), device="cuda", dtype=torch.float64)
C = torch.randn((jp, p), device="cuda", dtype=torch.float64)
for name, fn in (("tn", lambda: B.gemm(1, jp, V, C)), ("nn", lambda: B.gemm(0, jp, C, V, alpha=-1.0, beta=1.0))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"basis {name} jp={jp}: {ms*1e3:.1f} us; planes {7*n*jp/ms/1e6:.0f} GB/s", flush=True)
from torch.profiler import profile, ProfilerActivity
import collections
for name, fn in (("tn", lambda: B.gemm(1, jp, V, C)), ("nn", lambda: B.gemm(0, jp, C, V, alpha=-1.0, beta=1.0))):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
    agg = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name[:60]] += ev.device_time_total / 3.0
    print(name, {k: round(v, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])})
