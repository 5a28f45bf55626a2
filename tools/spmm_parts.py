"""C3 hybrid SpMM broken into its launches (torch profiler kernel times) and
a hot-density sweep. GPU only; prints one JSON object."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1504_05477_b200.operators import CsrDeviceOp  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def kernel_split(fn, reps=3):
    from torch.profiler import ProfilerActivity, profile

    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    out = {}
    for ev in prof.key_averages():
        if ev.device_type is not None and "cuda" in str(ev.device_type).lower() and ev.count:
            t = getattr(ev, "device_time_total", None) or getattr(ev, "cuda_time_total", 0)
            out[ev.key[:90]] = round(t / reps / 1e3, 4)
    return dict(sorted(out.items(), key=lambda kv: -kv[1]))


def main():
    cfgd = bench.CONFIGS["c3"]
    dev = torch.device("cuda", 0)
    indptr, col, val = bench.make_csr(cfgd, dev)
    n, d, p = cfgd["n"], cfgd["d"], cfgd["k"]
    g = torch.Generator(device=dev).manual_seed(5)
    X = torch.randn((d, p), generator=g, device=dev)
    Y = torch.randn((n, p), generator=g, device=dev)
    oy = torch.empty((n, p), device=dev)
    oc = torch.empty((d, p), device=dev)
    res = {"nnz": val.numel()}
    dens_list = [float(x) for x in os.environ.get("DENS", "0.03,0.015,0.008,0.06,0").split(",")]
    for dens in dens_list:
        op = CsrDeviceOp(indptr, col, val, d, hot_density=dens)
        leg = {"H": op.hot["H"] if op.hot else 0,
               "hot_nnz_frac": (op.hot["hot_nnz"] / val.numel()) if op.hot else 0.0,
               "slab_cols": int(op.slab["cols"].numel()) if op.slab else 0,
               "slab_nnz_frac": (op.slab["nnz"] / val.numel()) if op.slab else 0.0}
        leg["A.X_ms"] = timed(lambda: op.apply(X, oy))
        leg["A^T.Y_ms"] = timed(lambda: op.apply_t(Y, oc))
        if dens == dens_list[0]:
            leg["A.X_kernels_ms"] = kernel_split(lambda: op.apply(X, oy))
            leg["A^T.Y_kernels_ms"] = kernel_split(lambda: op.apply_t(Y, oc))
        res[f"dens_{dens}"] = leg
        del op
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
