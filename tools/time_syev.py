"""Time syev_topk on Rayleigh-Ritz-like matrices."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops
SH = [(200, 20), (600, 50), (1200, 200), (1600, 200)]
if len(sys.argv) > 1:
    SH = [tuple(int(x) for x in sys.argv[1].split(','))]
for w, k in SH:
    rng = np.random.default_rng(w)
    Q, _ = np.linalg.qr(rng.standard_normal((w, w)))
    lam = (np.arange(1, w + 1) ** -0.5) ** 2
    s = (Q * lam) @ Q.T
    M = torch.from_numpy(0.5 * (s + s.T)).cuda()
    ts = []
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        ev, E, info = ops.syev_topk(M, k)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    print(f"w={w} k={k}: {min(ts)*1e3:.2f} ms info={int(info[0])}", flush=True)
