"""Kernel-level timeline of one C2 exact-mode factorization replayed as a CUDA
graph (torch profiler / CUPTI): per-stream busy time, idle gaps on the union
of the streams, top kernels, and the launch sequence with start / duration
(gpurun_out/c2_graph_trace.csv). GPU only; profiler numbers are not bench
numbers."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import bench
from paper_1504_05477_b200 import matrix as mx
from paper_1504_05477_b200 import rsvd
from paper_1504_05477_b200.operators import DenseDeviceOp

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
cfgd = bench.CONFIGS[name]
cfg = rsvd.RsvdConfig(k=cfgd["k"], variant=cfgd["variant"], q=cfgd["q"], seed=0)
if cfgd.get("sparse"):
    from paper_1504_05477_b200.operators import CsrDeviceOp

    indptr, colv, valv = bench.make_csr(cfgd, torch.device("cuda", 0))
    op = CsrDeviceOp(indptr, colv, valv, cfgd["d"])
else:
    A = bench.make_matrix(cfgd, torch.device("cuda", 0))
    if cfgd.get("fp64") or mode == "fp64":
        A = A.double()
    op = DenseDeviceOp(A, exact=(mode == "exact"), center=bool(cfgd.get("pca")))
Pi = mx.gaussian(cfgd["d"], cfg.p, mx.SeededRng(0)).data
g = rsvd.GraphedFactorization(op, cfg)
for _ in range(3):
    g.run(Pi)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.run(Pi)
    torch.cuda.synchronize()
evs = []
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and ev.device_time_total > 0:
        evs.append((ev.time_range.start, ev.time_range.end, ev.name, getattr(ev, "device_resource_id", 0)))
evs.sort()


def short(nm):
    nm = nm.replace("(anonymous namespace)::", "").replace("void ", "").replace("rsvd::", "")
    return nm.split("(")[0][:70]


t0 = evs[0][0]
t1 = max(e[1] for e in evs)
print(f"span {(t1 - t0) / 1e3:.3f} ms, {len(evs)} device activities")
by_stream = collections.defaultdict(float)
by_name = collections.defaultdict(lambda: [0.0, 0])
for s, e, nm, st in evs:
    by_stream[st] += e - s
    k = short(nm)
    by_name[k][0] += e - s
    by_name[k][1] += 1
print("busy per stream (ms):", {k: round(v / 1e3, 3) for k, v in by_stream.items()})
# union busy / idle
busy = 0.0
cur_s, cur_e = evs[0][0], evs[0][1]
gaps = []
for s, e, nm, st in evs[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, cur_e - t0, nm))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"union busy {busy / 1e3:.3f} ms, idle {(t1 - t0 - busy) / 1e3:.3f} ms in {len(gaps)} gaps")
print("top kernels (ms, count):")
for k, (t, c) in sorted(by_name.items(), key=lambda kv: -kv[1][0])[:28]:
    print(f"  {t / 1e3:8.3f} {c:5d}  {k}")
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/{name}_graph_trace.csv", "w") as f:
    f.write("start_us,dur_us,stream,name\n")
    for s, e, nm, st in evs:
        f.write(f"{s - t0:.1f},{e - s:.1f},{st},{short(nm)}\n")
