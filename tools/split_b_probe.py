"""Gram through the tcgen05 path (split_b + TN + reduce) at C4 / C2 block shapes. Debug tool."""
import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_1504_05477_b200 import device as ops
g = torch.Generator(device="cuda").manual_seed(0)
for n, p in ((1000000, 200), (200000, 100)):
    V = torch.randn(n, p, generator=g, device="cuda")
    G = torch.empty(p, p, dtype=torch.float64, device="cuda")
    for _ in range(3): ops.gram(V, G, algo=2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): ops.gram(V, G, algo=2)
    e1.record(); torch.cuda.synchronize()
    ref = (V.double().T @ V.double())
    print(n, p, "gram (split_b + TN + reduce)", e0.elapsed_time(e1) / 10, "ms; rel err", float((G - ref).abs().max() / ref.abs().max()))
