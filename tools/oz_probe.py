"""Ozaki int8 products at the C2 shapes (A 50000 x 10000 FP32): NN width p,
TN width p; per-kernel device times from the torch profiler (for ncu captures
use -k k_oz_gemm). RSVD_OZ_ABLATE=1 no B loads, 2 no A loads, 4 no MMAs (sums
allowed). GPU only; not a bench number."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_1504_05477_b200 import device as ops

n, d = 50000, 10000
p = int(sys.argv[1]) if len(sys.argv) > 1 else 50
which = sys.argv[2] if len(sys.argv) > 2 else "both"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
plain = len(sys.argv) > 4 and sys.argv[4] == "plain"  # no CUPTI profiler (for runs under ncu)
A = torch.randn((n, d), device="cuda")
P = ops.OzPlanes(A)
X = torch.randn((d, p), device="cuda", dtype=torch.float64)
Y = torch.randn((n, p), device="cuda", dtype=torch.float64)
C = torch.empty((n, p), device="cuda", dtype=torch.float64)
W = torch.empty((d, p), device="cuda", dtype=torch.float64)
nplanes = int(ops.lib().rsvd_oz_num_planes())
for name, fn in (("nn", lambda: ops.oz_gemm(P, X, C, 0)), ("tn", lambda: ops.oz_gemm(P, Y, W, 1))):
    if which not in ("both", name):
        continue
    fn()
    torch.cuda.synchronize()
    if plain:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} p={p}: {e0.elapsed_time(e1) / reps:.3f} ms per product (all kernels)", flush=True)
        continue
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    agg = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name.split("<")[0].split("::")[-1][:24]] += ev.device_time_total / reps / 1e3
    g = agg.get("k_oz_gemm", 0.0)
    print(f"{name} p={p} ablate={os.environ.get('RSVD_OZ_ABLATE', '0')}: k_oz_gemm {g:.3f} ms "
          f"({nplanes * n * d / g / 1e6:.0f} GB/s of A planes); all: "
          + ", ".join(f"{k} {v:.3f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])), flush=True)
