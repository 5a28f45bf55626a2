"""Column sums of squares of an n x p FP32 block (C4 / C2 shapes). Debug tool."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
g = torch.Generator(device="cuda").manual_seed(0)
for n, p in ((1000000, 200), (50000, 50)):
    V = torch.randn(n, p, generator=g, device="cuda")
    out = torch.empty(p, dtype=torch.float64, device="cuda")
    for _ in range(3): ops.colreduce(V, True, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): ops.colreduce(V, True, out)
    e1.record(); torch.cuda.synchronize()
    ref = V.double().pow(2).sum(0)
    print(n, p, f"colreduce {e0.elapsed_time(e1) / 10 * 1e3:.1f} us; rel err {float(((out - ref) / ref).abs().max()):.2e}")
