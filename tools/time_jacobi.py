"""Time the device Jacobi (scalar vs block) on Rayleigh-Ritz-like matrices."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_05477_b200 import device as ops

def case(w, kind):
    rng = np.random.default_rng(w)
    Q, _ = np.linalg.qr(rng.standard_normal((w, w)))
    if kind == "decay":
        lam = (np.arange(1, w + 1) ** -0.5) ** 2
    else:
        lam = rng.standard_normal(w)
    s = (Q * lam) @ Q.T
    return 0.5 * (s + s.T)

for w in [int(x) for x in (sys.argv[1:] or ["200", "600", "1200", "1600"])]:
    for kind in ("decay",):
        sym = torch.from_numpy(case(w, kind)).cuda()
        for mode in ("block", "scalar"):
            if mode == "scalar":
                os.environ["RSVD_SCALAR_JACOBI"] = "1"
            else:
                os.environ.pop("RSVD_SCALAR_JACOBI", None)
            ts = []
            for rep in range(2):
                M = sym.clone(); V = torch.eye(w, dtype=torch.float64, device="cuda")
                torch.cuda.synchronize(); t = time.perf_counter()
                info, off = ops.jacobi_sweeps(M, V, 1e-14, 50)
                torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
            print(f"w={w} {kind} {mode}: {min(ts)*1e3:.2f} ms sweeps={int(info[1])} conv={int(info[0])}", flush=True)
