"""Timing of the orthonormalization-sized products (C2: n = 50000, p = 50)
through each GEMM algorithm. GPU only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops
from paper_1504_05477_b200.krylov import rows_buffer

def t(fn, reps=20):
    """GPU time per call: `reps` calls captured in a CUDA graph and replayed
    (the factorization runs as a graph, so host launch cost is not counted)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1e3

n, p = 50000, 50
g = torch.Generator(device="cuda").manual_seed(0)
X = rows_buffer(n, p, torch.float32, "cuda"); X.copy_(torch.randn(n, p, generator=g, device="cuda"))
Y = rows_buffer(n, p, torch.float32, "cuda")
T = torch.randn(p, p, generator=g, device="cuda")
G = torch.empty(p, p, dtype=torch.float64, device="cuda")
for w in (0, 100, 300, 550):
    if w:
        Qp = rows_buffer(n, w, torch.float32, "cuda"); Qp.copy_(torch.randn(n, w, generator=g, device="cuda"))
        C = torch.empty(w, p, dtype=torch.float32, device="cuda")
    for algo, name in ((4, "skinny"), (1, "simt"), (2, "tc")):
        if w == 0:
            a = t(lambda: ops.gemm_nn(X, T, Y, algo=algo))
            b = t(lambda: ops.gram(X, G, algo=algo))
            print(f"{name:6s} NN X.T (K={p}) {a:7.1f} us   gram X^T X -> f64 {b:7.1f} us")
        else:
            a = t(lambda: ops.gemm_tn(Qp, X, C, algo=algo))
            b = t(lambda: ops.gemm_nn(Qp, C, Y, alpha=-1.0, beta=1.0, algo=algo))
            print(f"{name:6s} w={w}: Qp^T X {a:7.1f} us   X -= Qp C (K={w}) {b:7.1f} us")
