"""GPU time of one chol_deflate at p (graph-replayed; host launch cost not
counted) and an ncu-friendly single launch. GPU only."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
for p in [int(x) for x in (sys.argv[1:] or ["50", "200"])]:
    rng = np.random.default_rng(0)
    v = rng.standard_normal((2000, p))
    G = torch.from_numpy(v.T @ v).cuda()
    T = torch.empty((p, p), dtype=torch.float64, device="cuda")
    mask = torch.empty(p, dtype=torch.int32, device="cuda")
    ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
    fn = lambda: ops.chol_deflate(G, None, 1e-14, T, mask, ndef)
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    print(f"chol_deflate p={p}: {e0.elapsed_time(e1)/100*1e3:.1f} us per call (graph)")
