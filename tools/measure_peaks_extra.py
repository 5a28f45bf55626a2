"""Measured tensor-core peaks that MEASURED_PEAKS.json lacks, taken the same
way the driver takes its bf16 figure (a cuBLAS GEMM, 8192^3, best of 10 with
CUDA events): TF32 (FP32 with allow_tf32), INT8 (torch._int_mm, int32
accumulate) and FP64 (DGEMM on the DMMA pipe). The 3xTF32 kernels are judged
against TF32 / 3, the Ozaki digit-plane kernels against the INT8 figure, the
DMMA kernels against FP64. Writes one JSON line."""
import json, sys
import torch


def best(fn, flops, reps=10):
    fn(); torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    ms = min(t)
    return flops / ms / 1e9, ms


n = 8192
out = {"gpu": torch.cuda.get_device_name(0), "how": "cuBLAS 8192^3 via torch, best of 10, CUDA events"}
a = torch.randn((n, n), device="cuda"); b = torch.randn((n, n), device="cuda")
torch.backends.cuda.matmul.allow_tf32 = True
out["tf32_tflops"], _ = best(lambda: a @ b, 2.0 * n ** 3)
torch.backends.cuda.matmul.allow_tf32 = False
out["fp32_simt_tflops"], _ = best(lambda: a @ b, 2.0 * n ** 3, reps=3)
a8 = torch.randint(-64, 65, (n, n), device="cuda", dtype=torch.int8)
b8 = torch.randint(-64, 65, (n, n), device="cuda", dtype=torch.int8).t().contiguous().t()
try:
    out["int8_tops"], _ = best(lambda: torch._int_mm(a8, b8), 2.0 * n ** 3)
except Exception as exc:  # noqa: BLE001
    out["int8_tops"] = None
    out["int8_error"] = repr(exc)[:200]
a64, b64 = a.double(), b.double()
out["fp64_tflops"], _ = best(lambda: a64 @ b64, 2.0 * n ** 3, reps=5)
print(json.dumps(out), flush=True)
