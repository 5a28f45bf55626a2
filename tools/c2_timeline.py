"""Where the C2 exact-mode factorization spends its time: CUDA events on
the main (chain) and side (final orthonormalization) streams around each
phase of one eager run, printed as a timeline (ms since start). GPU only."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1504_05477_b200 import rsvd, krylov, matrix as mx
from paper_1504_05477_b200.operators import DenseDeviceOp

cfgd = bench.CONFIGS["c2"]
cfg = rsvd.RsvdConfig(k=cfgd["k"], variant=cfgd["variant"], q=cfgd["q"], seed=0)
A = bench.make_matrix(cfgd, "cuda")
op = DenseDeviceOp(A, exact=True)
Pi = mx.gaussian(A.shape[1], cfg.p, mx.SeededRng(0)).data
for _ in range(2):
    rsvd.run_device(op, cfg, Pi=Pi)
torch.cuda.synchronize()
marks = []


def mark(label):
    e = torch.cuda.Event(enable_timing=True)
    e.record()  # current stream (main or side inside its context)
    marks.append((label, torch.cuda.current_stream().cuda_stream, e))


orig_orth = krylov.orth_block
def orth(*a, **k):
    qp = k.get("Qp")
    lab = "final" if k.get("basis", None) is not None or k.get("deflation_count") is not None else "chain-orth"
    mark(lab + "+")
    r = orig_orth(*a, **k)
    mark(lab + "-")
    return r
krylov.orth_block = orth
for name in ("apply", "apply_t"):
    f = getattr(op, name)
    def w(*a, _f=f, _n=name, **k):
        mark(_n + "+"); r = _f(*a, **k); mark(_n + "-"); return r
    setattr(op, name, w)
orig_rr = krylov.rayleigh_ritz
def rr(*a, **k):
    mark("rr+"); r = orig_rr(*a, **k); mark("rr-"); return r
krylov.rayleigh_ritz = rr
rsvd.krylov.rayleigh_ritz = rr
mark("start")
df = rsvd.run_device(op, cfg, Pi=Pi)
mark("end")
torch.cuda.synchronize()
t0 = marks[0][2]
main = marks[0][1]
agg = {}
open_ = {}
for lab, st, e in marks:
    t = t0.elapsed_time(e)
    key = ("main" if st == main else "side") + ":" + lab.rstrip("+-")
    if lab.endswith("+"):
        open_[key] = t
    elif lab.endswith("-") and key in open_:
        agg[key] = agg.get(key, 0.0) + t - open_.pop(key)
    print(f"{t:8.2f} {'M' if st == main else 'S'} {lab}")
print({k: round(v, 2) for k, v in agg.items()})
