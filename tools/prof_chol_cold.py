"""chol_deflate time when its code is cold (an L2-evicting write between
calls, as the Krylov chain's 2 GB stream does in a factorization) vs warm.
Debug tool:  python tools/prof_chol_cold.py [p ...]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops

big = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def graph_time(fn, reps=20):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (3 * reps) * 1e3


for p in [int(x) for x in (sys.argv[1:] or ["50"])]:
    rng = np.random.default_rng(0)
    v = rng.standard_normal((2000, p))
    G = torch.from_numpy(v.T @ v).cuda()
    T = torch.empty((p, p), dtype=torch.float64, device="cuda")
    mask = torch.empty(p, dtype=torch.int32, device="cuda")
    ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
    chol = lambda: ops.chol_deflate(G, None, 1e-14, T, mask, ndef)
    flush = lambda: big.fill_(1.0)
    warm = graph_time(chol)
    fl = graph_time(flush)
    both = graph_time(lambda: (flush(), chol()))
    print(f"p={p}: warm {warm:.1f} us, cold {both - fl:.1f} us (flush alone {fl:.1f} us)", flush=True)
