"""Time the FP32 3xTF32 tall-skinny products at a config's chain shape
(random operands; GPU only). Usage: gemm_probe.py [n d b reps]
Prints ms and algorithmic TFLOP/s (2 n d b) for A.X (NN) and A^T.Y (TN)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1504_05477_b200 import device as ops

n, d, b = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1000000, 4096, 200)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((n, d), generator=g, device="cuda")
X = torch.randn((d, b), generator=g, device="cuda")
Y = torch.randn((n, b), generator=g, device="cuda")
out_y = torch.empty((n, b), device="cuda")
out_x = torch.empty((d, b), device="cuda")
fl = 2.0 * n * d * b
for name, fn in (("NN A.X", lambda: ops.gemm_nn(A, X, out_y)), ("TN A^T.Y", lambda: ops.gemm_tn(A, Y, out_x))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name} n={n} d={d} b={b}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s", flush=True)
# accuracy spot check against FP64
rows = slice(0, 4096)
ref = (A[rows].double() @ X.double())
err = ((out_y[rows].double() - ref).abs().max() / ref.abs().max()).item()
ref_t = A.double().T @ Y.double() if n * d <= 2e8 else None
print(f"NN max rel err (first 4096 rows) {err:.2e}")
if ref_t is not None:
    print(f"TN max rel err {((out_x.double() - ref_t).abs().max() / ref_t.abs().max()).item():.2e}")
if os.environ.get("PROBE_PROFILE"):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ops.gemm_nn(A, X, out_y); ops.gemm_tn(A, Y, out_x); torch.cuda.synchronize()
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            print(f"  {ev.device_time_total / 1e3:8.3f} ms  {ev.name[:90]}")
