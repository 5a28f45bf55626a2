"""Per-index parity of the C2 factorization against the FP64 oracle (GPU +
~15 s of host oracle). Prints the worst indices and the deflation count."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import bench, rsvd_oracle as o
from paper_1504_05477_b200 import rsvd, matrix as mx
from paper_1504_05477_b200.operators import DenseDeviceOp
cfgd = bench.CONFIGS["c2"]
A = bench.make_matrix(cfgd, "cuda")
cfg = rsvd.RsvdConfig(k=cfgd["k"], variant=cfgd["variant"], q=cfgd["q"], seed=0)
Pi = mx.gaussian(A.shape[1], cfg.p, mx.SeededRng(0)).data
df = rsvd.run_device(DenseDeviceOp(A), cfg, Pi=Pi)
sig = df.sigma.cpu().numpy(); Z = df.Z
print("deflated columns:", None if df.deflated is None else int(df.deflated.sum()))
A64h = A.double().cpu().numpy()
r = o.factorize(o.DenseOp(A64h), cfg.k, "bk", q=cfg.q, p=cfg.p, seed=0)
rel = np.abs(sig - r.sigma) / r.sigma
A64 = A.double()
cap = (A64.T @ Z.double()).pow(2).sum(0).cpu().numpy()
cap_ref = (A64.T @ torch.from_numpy(np.ascontiguousarray(r.Z)).cuda()).pow(2).sum(0).cpu().numpy()
crel = np.abs(cap - cap_ref) / cap_ref
print("oracle deflated:", getattr(r, "deflated", "?"))
for i in np.argsort(-rel)[:6]:
    print(f"i={i:2d} sigma {sig[i]:.9f} ref {r.sigma[i]:.9f} rel {rel[i]:.2e}  cap rel {crel[i]:.2e}")
print("sigma tail ref:", np.round(r.sigma[40:], 6))
# exact singular values: sigma_i = sqrt(lambda_i(A^T A)), FP64 on the GPU
Gm = A64.T @ A64
ev = torch.linalg.eigvalsh(Gm).flip(0)[: cfg.k].clamp_min(0).sqrt().cpu().numpy()
del Gm
e_ours = np.abs(sig - ev) / ev
e_ref = np.abs(r.sigma - ev) / ev
print(f"vs exact SVD: ours max {e_ours.max():.2e} median {np.median(e_ours):.2e}; "
      f"reference max {e_ref.max():.2e} median {np.median(e_ref):.2e}")
print(f"ours >= reference for {(sig >= r.sigma - 1e-15).sum()} of {cfg.k}; ours <= exact (+1e-12) for "
      f"{(sig <= ev * (1 + 1e-12)).sum()} of {cfg.k}")
for i in (0, 10, 30, 38, 40, 47, 48, 49):
    print(f"i={i:2d} exact {ev[i]:.9f} ours {sig[i]:.9f} ({e_ours[i]:.1e}) ref {r.sigma[i]:.9f} ({e_ref[i]:.1e})")
# our FP64 path with the projected construction (near exact-arithmetic Krylov)
os.environ["RSVD_BK_BASIS"] = "projected"
from paper_1504_05477_b200 import krylov
krylov.BK_BASIS = "projected"
df64 = rsvd.run_device(DenseDeviceOp(A64), cfg, Pi=Pi)
s64 = df64.sigma.cpu().numpy()
krylov.BK_BASIS = "faithful"
df64f = rsvd.run_device(DenseDeviceOp(A64), cfg, Pi=Pi)
s64f = df64f.sigma.cpu().numpy()
f = lambda a, b: np.max(np.abs(a - b) / b)
print(f"FP64 projected vs reference {f(s64, r.sigma):.2e}; FP32 projected vs FP64 projected {f(sig, s64):.2e}; "
      f"FP64 faithful (ours) vs reference {f(s64f, r.sigma):.2e}")
# spectral error ||A - Z Z^T A||_2 (reference estimator, GPU): ours vs the reference's Z
import paper_1504_05477_b200 as rk
from paper_1504_05477_b200.operators import DenseDeviceOp as _D
op32 = _D(A)
from paper_1504_05477_b200 import metrics as M
mi = 5000
b_ours, it_o = M.spectral_norm_batched(M._Deflated(op32, M._as_device_z(Z, op32)), max_iters=mi)
b_ref, it_r = M.spectral_norm_batched(M._Deflated(op32, M._as_device_z(np.ascontiguousarray(r.Z), op32)), max_iters=mi)
so, sr = float(b_ours.max()), float(b_ref.max())
print(f"spectral error (<= {mi} power iterations per start, FP32 A): ours {so:.9f} reference Z {sr:.9f} rel {abs(so-sr)/sr:.2e}; iterations {it_o.tolist()} / {it_r.tolist()}")
