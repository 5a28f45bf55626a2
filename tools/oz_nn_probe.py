import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_1504_05477_b200 import device as ops
from torch.profiler import profile, ProfilerActivity
import collections
n, w, p = 50000, 600, 50
jp = 300
Q = torch.randn((n, w), device="cuda", dtype=torch.float64) / n ** 0.5
B = ops.OzBasis(n, w, Q.device)
for c0 in range(0, w, p):
    B.slice(Q, c0, p)
V = torch.randn((n, p), device="cuda", dtype=torch.float64)
V2 = torch.randn((n, 64), device="cuda", dtype=torch.float64)[:, :50]
Kview = torch.randn((n, 600), device="cuda", dtype=torch.float64)[:, 100:150]
C = torch.randn((jp, p), device="cuda", dtype=torch.float64)
tests = (("nn beta1 contiguous", lambda: B.gemm(0, jp, C, V, alpha=-1.0, beta=1.0)),
         ("nn beta0 contiguous", lambda: B.gemm(0, jp, C, V)),
         ("nn beta1 ld600 view", lambda: B.gemm(0, jp, C, Kview, alpha=-1.0, beta=1.0)),
         ("nn beta1 jp=50", lambda: B.gemm(0, 50, C[:50], V, alpha=-1.0, beta=1.0)))
for name, fn in tests:
    fn(); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
    agg = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA and "k_oz_gemm" in ev.name:
            agg["gemm"] += ev.device_time_total / 3.0
    print(name, dict(agg), flush=True)
