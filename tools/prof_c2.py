"""Kernel-time breakdown of one eager C2 factorization (torch.profiler, CUDA
activity), grouped by kernel name. GPU only; not a bench number."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1504_05477_b200 import rsvd, matrix as mx
from paper_1504_05477_b200.operators import DenseDeviceOp

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfgd = bench.CONFIGS[cfgname]
cfg = rsvd.RsvdConfig(k=cfgd["k"], variant=cfgd["variant"], q=cfgd["q"], seed=0)
n, d = cfgd["n"], cfgd["d"]
if cfgd.get("sparse"):
    from paper_1504_05477_b200.operators import CsrDeviceOp
    op = CsrDeviceOp(*bench.make_csr(cfgd, "cuda"), d)
else:
    A = bench.make_matrix(cfgd, "cuda")
    op = DenseDeviceOp(A, n_total=n, row_offset=0)
Pi = mx.gaussian(d, cfg.p, mx.SeededRng(cfg.seed)).data
for _ in range(2):
    rsvd.run_device(op, cfg, Pi=Pi)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rsvd.run_device(op, cfg, Pi=Pi)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        nm = ev.name
        nm = nm[5:] if nm.startswith("void ") else nm
        nm = nm.replace("rsvd::(anonymous namespace)::", "").replace("rsvd::", "")
        depth = 0
        for i, ch in enumerate(nm):
            depth += ch == "<"
            depth -= ch == ">"
            if ch == "(" and depth == 0:
                nm = nm[:i]
                break
        name = nm[:80]
        agg[name][0] += ev.device_time_total / 1e3 if hasattr(ev, "device_time_total") else ev.cuda_time_total / 1e3
        agg[name][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"total kernel time {tot:.2f} ms over {sum(v[1] for v in agg.values())} kernels")
for name, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{t:8.3f} ms {100*t/tot:5.1f}% x{c:4d}  {name}")
