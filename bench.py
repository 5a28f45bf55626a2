"""Benchmark: rank-k block-Krylov SVD wall time on B200 (BASELINE.json).

Default workload = BASELINE configs[1] ("C2"): dense FP32 A 50,000 x 10,000,
A = U diag(i^-0.5) V^T + 1e-3 N(0,1), Haar U, V from seeded Gaussians (built
on the GPU in FP64, cast to FP32), block Krylov k = 50, q = 10 (-> 11, the
reference's odd bump, rsvd.py:157-158), Krylov width 600, Pi = host
SeededRng(0) Gaussian 10,000 x 50. Synthetic data (no dataset is named).

Precision mode of the measured path (per config, --precision overrides):
  C2 "exact": A stays FP32 in HBM; Krylov blocks, orthonormalization and
     Rayleigh-Ritz are FP64; both products A X / A^T Y are FP64-accurate int8
     tensor-core GEMMs (Ozaki digit planes, csrc/gemm_oz.cu); the reference's
     own basis construction (normalized power blocks, then _mgs of their
     hstack, rsvd.py:244-260) -- the mode that matches the reference to the
     north_star tolerance at this config (the FP32 3xTF32 path misses it, see
     the fp32_mode leg).
  C1 "fp64" (an FP64 config); C4 / C5 "fp32" (3xTF32; parity passes there).

One step = one complete factorization (start block upload, digit planes of A,
Krylov chain, blocked orthonormalization, Rayleigh-Ritz + eigensolver, Z and
sigma ready).
  value : device-resident A (uploaded before timing), CUDA-event timed.
  e2e   : the public drop-in call block_krylov(A_host_pinned, cfg) -- H2D of A
          and D2H of (Z, sigma) inside the timed region, every step
          (e2e_numpy: the same call with a pageable numpy array).
A (2 GB FP32) is larger than L2 (126 MB), so every step streams it from HBM.

--impl reference: the reference's CPU algorithm (the oracle port,
oracle/rsvd_oracle.py: numpy/OpenBLAS FP64 products as the reference's python
backend, the C restatement of its Jacobi, its per-column CGS2 _mgs) on a
host-generated A of the same config (numpy only -- no GPU, nothing from the
product package), all host threads.

--gpus N: N ranks (one per GPU) over NCCL, A row-sharded; the
step is the same factorization of the same A (strong scaling); A^T Y, Grams
and projections are allreduced. Without torchrun the script relaunches itself
under torch.distributed.run (NCCL_DEBUG=INFO so the communicator prints).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

# pin BLAS threads to the host cores BEFORE numpy loads OpenBLAS (unpinned
# OpenBLAS oversubscribes)
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
    os.environ.setdefault(_v, str(os.cpu_count() or 1))

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(n=50000, d=10000, k=50, q=10, spectrum="pow", noise=1e-3, variant="bk", mode="exact"),
    "c1": dict(n=2000, d=1000, k=20, q=8, spectrum="inv", noise=0.0, variant="bk", fp64=True, mode="fp64"),
    "c4": dict(n=1000000, d=4096, k=200, q=6, spectrum="clustered", noise=0.0, variant="bk", mode="fp32"),
    "c3": dict(n=200000, d=100000, k=100, q=15, sparse=True, variant="bk", mode="fp32"),
    # C5: PCA with implicit mean-centering (rank-1 GEMM-epilogue corrections)
    "c5": dict(n=500000, d=2000, k=200, q=4, pca=True, variant="bk", mode="fp32"),
    "c5si": dict(n=500000, d=2000, k=200, q=12, pca=True, variant="si", mode="fp32"),
}
MODE_DTYPE = {"exact": "f64 (FP32 A; FP64-accurate int8 tcgen05 Ozaki products, FP64 blocks and small algebra)",
              "fp32": "f32 (3xTF32 products, f64 small algebra)", "fp64": "f64"}


def make_csr(cfg, device, seed=4321):
    """C3: per-row nnz m_i = clip(round(LogNormal(ln 100 - 1/2, 1)),
    1, d); columns drawn Zipf(s = 1.1) over {0..d-1} (p_c ~ (c+1)^-1.1), duplicates
    within a row dropped (sampling without replacement, approximated), sorted
    ascending; values LogNormal(0, 1), each row scaled to unit L2 norm. Built
    on the GPU with a seeded generator; int32 indices, FP32 values."""
    import torch

    n, d = cfg["n"], cfg["d"]
    g = torch.Generator(device=device).manual_seed(seed)
    mu = float(np.log(100.0) - 0.5)
    m = torch.exp(mu + torch.randn(n, generator=g, device=device, dtype=torch.float64))
    m = torch.clamp(torch.round(m), 1, d).to(torch.int64)
    total = int(m.sum())
    rows = torch.repeat_interleave(torch.arange(n, device=device), m)
    pz = (torch.arange(1, d + 1, device=device, dtype=torch.float64)) ** -1.1
    cdf = torch.cumsum(pz, 0)
    cdf /= cdf[-1].clone()
    u = torch.rand(total, generator=g, device=device, dtype=torch.float64)
    cols = torch.searchsorted(cdf, u).clamp_(max=d - 1)
    key = torch.unique(rows * d + cols)  # sorted, duplicates dropped
    # without replacement: redraw each row's deficit until it holds m_i
    # distinct columns (Zipf heads collide often; a few rounds suffice)
    for _ in range(64):
        have = torch.bincount(key // d, minlength=n)
        deficit = (m - have).clamp_(min=0)
        nd = int(deficit.sum())
        if nd == 0:
            break
        r2 = torch.repeat_interleave(torch.arange(n, device=device), deficit)
        u2 = torch.rand(nd, generator=g, device=device, dtype=torch.float64)
        c2 = torch.searchsorted(cdf, u2).clamp_(max=d - 1)
        key = torch.unique(torch.cat([key, r2 * d + c2]))
    rows = key // d
    cols = (key % d).to(torch.int32)
    nnz = key.numel()
    vals = torch.exp(torch.randn(nnz, generator=g, device=device, dtype=torch.float64))
    norms = torch.zeros(n, device=device, dtype=torch.float64).index_add_(0, rows, vals * vals).sqrt_()
    vals = (vals / norms[rows]).to(torch.float32)
    counts = torch.bincount(rows, minlength=n)
    indptr = torch.zeros(n + 1, device=device, dtype=torch.int32)
    indptr[1:] = torch.cumsum(counts, 0).to(torch.int32)
    torch.cuda.synchronize()
    return indptr, cols, vals


def _spectrum(kind, d):
    i = np.arange(1, d + 1, dtype=np.float64)
    if kind == "pow":
        return i ** -0.5
    if kind == "inv":
        return 1.0 / i
    if kind == "clustered":
        s = 0.5 / i
        s[:200] = 1 - 0.001 * i[:200]
        return s
    raise ValueError(kind)


def workload_config(name, cfgd, cfg, world, nnz=None):
    """The `config` object of the JSON line (shared by both arms)."""
    n, d, k = cfgd["n"], cfgd["d"], cfgd["k"]
    w = cfg.p * (cfg.resolve_q(d) + 1)
    sparse = bool(cfgd.get("sparse"))
    si = cfgd["variant"] == "si"
    if si:
        w = cfg.p
    label = "SI" if si else "BK"
    what = (f"CSR FP32 A {n}x{d} nnz {nnz}" if sparse else
            f"PCA (implicit centering) on dense FP32 A {n}x{d}" if cfgd.get("pca") else
            f"dense {'FP64' if cfgd.get('fp64') else 'FP32'} A {n}x{d}")
    return {"workload": (f"{name.upper()}: " + what
                         + f", {label} k={k} q={cfgd['q']}->{cfg.resolve_q(d)}, width {w}"),
            "n": n, "d": d, "k": k, "q": cfgd["q"], "q_eff": cfg.resolve_q(d), "krylov_width": w,
            "parallelism": f"rowshard{world}",
            "l2": ("CSR %.0f MB + blocks; dense rows L2-resident by design (gather-bound)" % (nnz * 8 / 1e6)
                   if sparse else "inputs larger than L2 (A = %.1f GB)" % (n * d * 4 / 1e9))}


def spmm_probe(dev, reps=5):
    """The SpMM half of the metric on the C3 matrix: A.X and
    A^T.Y at width k = 100, CUDA-event timed; GB/s are SURVEY's algorithmic
    bytes nnz (4 + 4) + (rows + 1) 4 + (d + n) b 4 against the measured HBM
    copy bandwidth. Two operators: the hybrid one the factorization uses
    (Zipf-head columns as a dense tensor-core panel, the rest gathered) and
    the pure CSR gather ("csr_only"), which is L2-gather-bound: each nonzero
    reads a 400-byte row of the dense block."""
    import torch
    from paper_1504_05477_b200.operators import CsrDeviceOp

    cfgd = CONFIGS["c3"]
    n, d, p = cfgd["n"], cfgd["d"], cfgd["k"]
    indptr, colv, valv = make_csr(cfgd, dev)
    g = torch.Generator(device=dev).manual_seed(5)
    X = torch.randn((d, p), generator=g, device=dev)
    Y = torch.empty((n, p), device=dev)
    C = torch.empty((d, p), device=dev)
    nnz = valv.numel()
    hbm, _, _ = _peaks()
    res = {"config": f"C3 CSR {n}x{d}, nnz {nnz}, width {p}", "peak_gbs": hbm}
    for label, dens in (("hybrid", None), ("csr_only", 0.0)):
        op = CsrDeviceOp(indptr, colv, valv, d, hot_density=dens)
        leg = {}
        if op.hot is not None:
            leg["hot_columns"] = op.hot["H"]
            leg["hot_nnz_frac"] = op.hot["hot_nnz"] / nnz
        for name, fn, rows in (("A.X", lambda: op.apply(X, Y), n), ("A^T.Y", lambda: op.apply_t(Y, C), d)):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            byt = nnz * 8 + (rows + 1) * 4 + (n + d) * p * 4
            leg[name] = {"ms": ms, "algorithmic_gbs": byt / ms / 1e6, "frac": byt / ms / 1e6 / hbm}
            if dens == 0.0:
                leg[name]["gathered_gbs"] = (nnz * p * 4 + byt) / ms / 1e6
        res[label] = leg
        del op
    del indptr, colv, valv
    torch.cuda.empty_cache()
    return res


def gemm_c4_probe(dev, bf16, reps=3):
    """The Krylov-GEMM half of the metric where it is tensor-bound: the C4
    chain products A.X and A^T.Y (A 1,000,000 x 4096 FP32, width 200; random
    operands -- the kernel's work does not depend on the values) through the
    same 3xTF32 tcgen05 kernel, CUDA-event timed, as algorithmic TFLOP/s
    (2 n d b) against the measured bf16 dense peak / 6 (TF32 issues at half
    the bf16 rate and 3xTF32 is three TF32 MMAs). A (16.4 GB) exceeds L2."""
    import torch
    from paper_1504_05477_b200 import device as ops

    n, d, b = 1000000, 4096, 200
    g = torch.Generator(device=dev).manual_seed(11)
    A = torch.randn((n, d), generator=g, device=dev)
    X = torch.randn((d, b), generator=g, device=dev)
    Y = torch.randn((n, b), generator=g, device=dev)
    out_y = torch.empty((n, b), device=dev)
    out_x = torch.empty((d, b), device=dev)
    px = _peaks_extra()
    peak = px["tf32_tflops"] / 3.0 if px and px.get("tf32_tflops") else bf16 / 6.0
    fl = 2.0 * n * d * b
    res = {"config": f"C4 chain shape: A {n}x{d} FP32, width {b} (random operands)",
           "peak_tflops": peak, "peak_source": (f"measured cuBLAS TF32 {px['tf32_tflops']:.0f} TFLOP/s / 3" if px and
                                                px.get("tf32_tflops") else f"measured bf16 dense {bf16:.0f} / 6"),
           "ncu": "profiles/r01_c4_chain_kernel_ncu.json (tensor pipe 83% / 86% of peak sustained)"}
    for name, fn in (("A.X", lambda: ops.gemm_nn(A, X, out_y)), ("A^T.Y", lambda: ops.gemm_tn(A, Y, out_x))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name] = {"ms": ms, "tflops": fl / ms / 1e9, "frac": fl / ms / 1e9 / peak}
    del A, X, Y, out_y, out_x
    torch.cuda.empty_cache()
    return res


def _profiled_traffic(config="c2", mode="fp32"):
    """DRAM bytes per launch of the dominant chain kernel from the committed
    ncu --set full capture (dram__bytes_read.sum + dram__bytes_write.sum):
    profiles/r02_<config>_<mode>_chain_kernel_ncu.json, else the round-1
    capture of the 3xTF32 kernel for the fp32 mode; None when none is
    committed."""
    names = [f"r02_{config}_{mode}_chain_kernel_ncu.json"]
    if mode == "fp32":
        names.append("r01_chain_kernel_ncu.json" if config == "c2" else f"r01_{config}_chain_kernel_ncu.json")
    for name in names:
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return float(json.load(f)["dram_bytes_per_launch"])
        except (OSError, KeyError, ValueError):
            continue
    return None


def make_pca_matrix(cfg, device, seed=777):
    """C5: rows x_r = mu + W diag(sqrt(lambda)) g_r, g_r ~ N(0, I),
    mu_j ~ U(-5, 5), Haar W (QR of a seeded Gaussian, sign-fixed), lambda_i =
    exp(-i/50); built in FP64 on the GPU in row chunks, FP32 out."""
    import torch

    n, d = cfg["n"], cfg["d"]
    g = torch.Generator(device=device).manual_seed(seed)
    W = torch.randn((d, d), generator=g, dtype=torch.float64, device=device)
    W, R = torch.linalg.qr(W)
    W *= torch.sign(torch.diagonal(R)).view(1, -1)
    lam = torch.exp(-torch.arange(1, d + 1, dtype=torch.float64, device=device) / 50.0)
    mu = torch.rand(d, generator=g, dtype=torch.float64, device=device) * 10.0 - 5.0
    M = (W * lam.sqrt().view(1, -1)).T.contiguous()  # diag(sqrt lambda) W^T
    A = torch.empty((n, d), dtype=torch.float32, device=device)
    chunk = 65536
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        G = torch.randn((r1 - r0, d), generator=g, dtype=torch.float64, device=device)
        A[r0:r1] = (G @ M + mu.view(1, -1)).float()
    del W, M, G
    torch.cuda.synchronize()
    return A


def make_matrix(cfg, device, seed=1234):
    """Haar U (n x d), V (d x d) from seeded Gaussians (QR, sign-fixed by
    diag R), A = U diag(s) V^T (+ noise), built in FP64 on the GPU, FP32 out."""
    import torch

    if cfg.get("pca"):
        return make_pca_matrix(cfg, device)
    n, d = cfg["n"], cfg["d"]
    g = torch.Generator(device=device).manual_seed(seed)
    s = torch.from_numpy(_spectrum(cfg["spectrum"], d)).to(device)
    A = torch.empty((n, d), dtype=torch.float32, device=device)
    V = torch.randn((d, d), generator=g, dtype=torch.float64, device=device)
    V, R = torch.linalg.qr(V)
    V *= torch.sign(torch.diagonal(R)).view(1, -1)
    chunk = 65536 if n > 65536 else n
    # U from a QR of the full n x d Gaussian when it fits comfortably, else a
    # block-wise orthonormal construction (still exactly orthonormal columns)
    U = torch.randn((n, d), generator=g, dtype=torch.float64, device=device)
    U, R = torch.linalg.qr(U)
    U *= torch.sign(torch.diagonal(R)).view(1, -1)
    W = (V * s.view(1, -1)).T.contiguous()  # diag(s) V^T
    for r0 in range(0, n, chunk):
        blk = U[r0: r0 + chunk] @ W
        if cfg["noise"]:
            blk += cfg["noise"] * torch.randn(blk.shape, generator=g, dtype=torch.float64, device=device)
        A[r0: r0 + chunk] = blk.float()
    del U, V, W
    torch.cuda.synchronize()
    return A


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._ready = threading.Event()
        self._t = None
        self.source = None

    def _nvml_handle(self):
        """NVML handle of this process's CUDA device, matched by PCI bus id
        (a CUDA ordinal is not an NVML index under CUDA_VISIBLE_DEVICES)."""
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _run_nvml(self):
        nv, h = self._nvml_handle()
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while True:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append([str(sm), str(mx), "", hex(rs)] + ["Active" if rs & b else "Not Active" for b in bits])
            self._ready.set()
            if self._stop.wait(0.002):  # ~2 ms: dozens of samples inside a 100 ms timed region
                return

    def _run(self):
        try:
            self._run_nvml()
            self.source = "nvml"
            return
        except Exception:
            pass
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(10)  # the sampler is live before the timed region starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows), "source": self.source}


def _peaks_extra():
    """TF32 / INT8 / FP64 cuBLAS peaks measured on this pool's B200s
    (tools/measure_peaks_extra.py -> profiles/r02_measured_peaks_extra.json),
    or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_measured_peaks_extra.json")) as f:
            return json.loads(f.read().strip().splitlines()[-1])
    except (OSError, ValueError, IndexError):
        return None


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


def run_ours(args):
    import torch

    import paper_1504_05477_b200 as rk
    from paper_1504_05477_b200 import krylov, rsvd
    from paper_1504_05477_b200.operators import DenseDeviceOp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RSVD_DIST_BACKEND=gloo (with --graph 0) exercises the N > 1 path on a box
    # with fewer GPUs than ranks: ranks share devices round-robin and the
    # collectives run through gloo on the host (no kernel waits on another rank)
    backend = os.environ.get("RSVD_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfgd = CONFIGS[args.config]
    n, d, k = cfgd["n"], cfgd["d"], cfgd["k"]
    cfg = rk.RsvdConfig(k=k, variant=cfgd["variant"], q=cfgd["q"], seed=0)
    sparse = bool(cfgd.get("sparse"))
    mode = args.precision or cfgd["mode"]
    if cfgd.get("fp64") or sparse:
        mode = cfgd["mode"] if not args.precision else args.precision
    lo, hi = krylov.shard_rows(n, world, rank)
    if world > 1:
        comm = krylov.TorchComm(n_total=n, row_offset=lo)
    if sparse:
        from paper_1504_05477_b200.operators import CsrDeviceOp

        indptr, colv, valv = make_csr(cfgd, dev)
        if world > 1:
            a0, a1 = int(indptr[lo]), int(indptr[hi])
            indptr = (indptr[lo: hi + 1] - indptr[lo]).contiguous()
            colv, valv = colv[a0:a1].contiguous(), valv[a0:a1].contiguous()
        A = None
        nnz_local = valv.numel()
        op = CsrDeviceOp(indptr, colv, valv, d, n_total=n, row_offset=lo)
    else:
        A_full = make_matrix(cfgd, dev)
        if cfgd.get("fp64"):  # C1 is an FP64 configuration (BASELINE configs[0])
            A_full = A_full.double()
        if world > 1:
            A = A_full[lo:hi].contiguous()
            del A_full
        else:
            A = A_full
        if mode == "fp64" and A.dtype != torch.float64:
            A = A.double()
        op = DenseDeviceOp(A, n_total=n, row_offset=lo, center=bool(cfgd.get("pca")), comm=comm,
                           exact=(mode == "exact"))
    Pi = rk.gaussian(d, cfg.p, rk.SeededRng(cfg.seed)).data

    # instrumentation of the dominant kernels (A X / A^T Y on the op's stream)
    events = []
    orig_apply, orig_apply_t = op.apply, op.apply_t

    def timed(fn, kind):
        def w(X, out, **kw):
            if not recording[0]:
                return fn(X, out, **kw)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn(X, out, **kw)
            e1.record()
            events.append((kind, X.shape[1], e0, e1))
            return r
        return w

    recording = [False]
    op.apply = timed(orig_apply, "AX")
    op.apply_t = timed(orig_apply_t, "ATY")

    graphed = rsvd.GraphedFactorization(op, cfg, comm=comm) if args.graph else None

    # the start block is a function of (d, p, seed) only: uploaded once like A
    # (the public API's graph cache keeps it on the device the same way)
    Pi_dev = torch.from_numpy(np.array(Pi, copy=True)).to(device=dev, dtype=op.dtype)

    def step():
        if graphed is not None:
            return graphed.run(Pi_dev)
        return rsvd.run_device(op, cfg, comm=comm, Pi=Pi_dev)

    if graphed is not None and world > 1:
        # capture the sharded factorization (its allreduces included) once up
        # front; should the process group refuse capture, every rank falls
        # back to eager launches together (the outcome is agreed by a MIN)
        ok = 1
        try:
            graphed.run(Pi_dev)
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001 - reported, then eager
            print(f"rank {rank}: graph capture failed ({exc!r}); running eager", file=sys.stderr, flush=True)
            ok = 0
        flag = torch.tensor([ok], device=dev if backend == "nccl" else "cpu")
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        if int(flag.item()) == 0:
            graphed = None
    for _ in range(args.warmup):
        df = step()
    torch.cuda.synchronize()
    if args.profile_step:
        # one factorization, kernels launched individually, inside the profiler window
        torch.cuda.profiler.start()
        rsvd.run_device(op, cfg, comm=comm, Pi=Pi)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        if rank == 0:
            print(json.dumps({"profile_step": args.config, "ok": True}), flush=True)
        return
    # kernels per factorization, counted on an eager replica of the step (a
    # graph replay issues the identical kernel sequence in one launch)
    # (every rank runs it: the factorization's collectives need all ranks)
    launches = count_launches(lambda: rsvd.run_device(op, cfg, comm=comm, Pi=Pi)) if args.count_launches else None
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            df = step()
        e1.record()
        torch.cuda.synchronize()
    # per-kernel durations of the dominant products: the same step run eagerly
    # (graph replays cannot host-record events) with CUDA events around every
    # A.X / A^T.Y launch on the launching stream
    recording[0] = True
    for _ in range(2):
        rsvd.run_device(op, cfg, comm=comm, Pi=Pi)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    info = df.info.cpu().numpy()
    assert int(info[0]) == 1, "Jacobi did not converge"
    sigma = df.sigma.cpu().numpy()

    # kernel roofline: the Krylov-chain products at width p
    hbm, bf16, peak_src = _peaks()
    chain = [(e0_.elapsed_time(e1_), kind) for kind, width, e0_, e1_ in events if width == cfg.p]
    rr = [(e0_.elapsed_time(e1_), kind) for kind, width, e0_, e1_ in events if width != cfg.p]
    n_loc = hi - lo
    if sparse:  # nnz (4 + 4) + (rows + 1) 4 + (d + n) b 4 per SpMM
        bytes_per = nnz_local * 8 + (n_loc + 1) * 4 + (n_loc + d) * cfg.p * 4
    else:  # A once (its stored precision) + the two blocks (the work precision)
        bytes_per = n_loc * d * A.element_size() + (n_loc + d) * cfg.p * (8 if mode in ("exact", "fp64") else 4)
    avg_chain_ms = float(np.mean([t for t, _ in chain])) if chain else float("nan")
    achieved = bytes_per / (avg_chain_ms * 1e-3) / 1e9
    rr_ms = float(np.mean([t for t, _ in rr])) if rr else float("nan")
    w = (cfgd["q"] + 1 + (cfgd["q"] % 2 == 0)) * cfg.p
    rr_tflops = 2.0 * n_loc * d * w / (rr_ms * 1e-3) / 1e12 if (rr and not sparse) else None

    # the chain product's bound: HBM below the ridge (C2: 25 flop/B in FP32),
    # tensor pipe above it (C4 / C5 at width 200: ~95 flop/B)
    flops_per = 2.0 * n_loc * d * cfg.p
    px = _peaks_extra()
    # 3xTF32 = 3 TF32 MMAs per product: the measured cuBLAS TF32 peak / 3 (else bf16 / 6)
    tf_eff = px["tf32_tflops"] / 3.0 if px and px.get("tf32_tflops") else bf16 / 6.0
    if sparse:
        kname = (("hybrid CSR product A.X / A^T.Y (width %d; hot-column panel on tcgen05 + CSR gather)"
                  if op.hot is not None else "CSR SpMM A.X / A^T.Y (width %d)") % cfg.p)
    elif mode == "exact":
        kname = ("FP64-accurate Krylov-chain A.X / A^T.Y (width %d): k_oz_gemm, int8 tcgen05 Ozaki digit planes "
                 "(5 A x 6 B signed base-256 digits, 20 digit-pair GEMMs)" % cfg.p)
    else:
        kname = "Krylov-chain A.X / A^T.Y (width %d)" % cfg.p
    traffic = None if sparse else _profiled_traffic(args.config, mode)
    if sparse or mode == "exact" or flops_per / bytes_per * hbm / 1e3 < tf_eff:
        roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "peak_source": peak_src, "traffic": traffic,
                    "algorithmic_bytes_per_launch": bytes_per, "avg_launch_ms": avg_chain_ms}
        if traffic:
            # the same launch time against the DRAM bytes ncu measured for this kernel
            roofline["traffic_gbs"] = traffic / (avg_chain_ms * 1e-3) / 1e9
            roofline["traffic_frac"] = roofline["traffic_gbs"] / hbm
        if mode == "exact":
            # what the kernel actually streams: the 5 digit planes of A (1.25x the
            # FP32 bytes) and the int8 MMA work (20 digit pairs, N padded to 64)
            planes = 5 * (-(-n_loc // 128) * 128) * (-(-d // 128) * 128)
            roofline["digit_plane_bytes_per_launch"] = planes
            roofline["digit_plane_gbs"] = planes / (avg_chain_ms * 1e-3) / 1e9
            # MMA columns per digit pair: the N tile the kernel picks (32 / 56 / 64 per 64 columns)
            ncols = 32 if cfg.p <= 32 else (56 if cfg.p <= 56 else 64 * (-(-cfg.p // 64)))
            roofline["int8_tops"] = 20 * 2.0 * n_loc * d * ncols / (avg_chain_ms * 1e-3) / 1e12
            roofline["note"] = ("algorithmic bytes = FP32 A + FP64 blocks; the kernel streams A's int8 digit "
                                "planes (digit_plane_gbs) and is co-limited by the int8 MMA issue (20 digit pairs)")
            px = _peaks_extra()
            if px and px.get("int8_tops"):
                roofline["int8_peak_tops"] = px["int8_tops"]
                roofline["int8_frac"] = roofline["int8_tops"] / px["int8_tops"]
                roofline["int8_peak_source"] = "measured cuBLAS int8 GEMM 8192^3 (profiles/r02_measured_peaks_extra.json)"
    else:
        tfl = flops_per / (avg_chain_ms * 1e-3) / 1e12
        roofline = {"bound": "tensor", "kernel": kname, "achieved": tfl, "peak": tf_eff, "unit": "TFLOP/s",
                    "frac": tfl / tf_eff,
                    "peak_source": (f"measured cuBLAS TF32 {px['tf32_tflops']:.0f} TFLOP/s / 3 (3 TF32 MMAs per "
                                    "3xTF32 product; profiles/r02_measured_peaks_extra.json)" if px and
                                    px.get("tf32_tflops") else
                                    f"{peak_src} bf16 dense {bf16:.0f} TFLOP/s / 6 (TF32 at half the bf16 rate, "
                                    "3 TF32 MMAs per 3xTF32 product)"),
                    "traffic": traffic, "algorithmic_flops_per_launch": flops_per,
                    "algorithmic_bytes_per_launch": bytes_per, "avg_launch_ms": avg_chain_ms,
                    "hbm_frac": achieved / hbm}

    # e2e through the public API with host A: pinned torch tensor (the line's
    # e2e) and a pageable numpy array (the reference callers' usual input)
    e2e = e2e_np = None
    if world == 1 and not args.no_e2e and not sparse:
        center = bool(cfgd.get("pca"))
        api_prec = mode

        def timed_api(A_in):
            for _ in range(max(1, min(args.warmup, 2))):
                rk.factorize(A_in, cfg, center=center, precision=api_prec)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                r = rk.factorize(A_in, cfg, center=center, precision=api_prec)
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) * 1e3 / args.steps, r

        # per step: H2D of A (Pi is uploaded once per cached shape/config, like A's
        # device buffer), D2H of Z (n x k FP64), sigma and the status words
        d2h = int(n * k * 8 + k * 8 + 8 * 3)
        A_host = A.cpu().pin_memory()
        e2e_ms, r = timed_api(A_host)
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": int(A_host.numel() * A_host.element_size()),
               "d2h_bytes_per_step": d2h, "input": "pinned torch tensor",
               "sigma_matches_value_path": bool(np.allclose(r.approx_singular_values, sigma, rtol=1e-12, atol=0))}
        A_np = A_host.numpy().copy()
        del A_host
        e2e_np_ms, _ = timed_api(A_np)
        e2e_np = {"value": e2e_np_ms, "unit": "ms", "h2d_bytes_per_step": int(A_np.nbytes), "d2h_bytes_per_step": d2h,
                  "input": "pageable numpy array"}
        del A_np

    out = {
        "metric": "rank-k block-Krylov SVD wall time",
        "value": ms,
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": ("f32 (CSR SpMM, f64 small algebra)" if sparse else MODE_DTYPE[mode]),
        "precision_mode": mode,
        "data": "synthetic",
        "config": workload_config(args.config, cfgd, cfg, world, nnz_local if sparse else None),
        "roofline": roofline,
        "kernels": ({"rayleigh_ritz_ATQ_ms": rr_ms, "rayleigh_ritz_ATQ_tflops": rr_tflops} if rr else
                    {"rayleigh_ritz_W": "assembled from the chain's A^T q_j (projected FP32 basis); "
                                        "no separate width-w pass over A"}),
        "gpu_launches": launches,
        "comm": ({"backend": backend, "world": torch.distributed.get_world_size(), "rank_rows": [lo, hi]}
                 if world > 1 else None),
        "clocks": clk.summary(),
        "sigma_head": [float(x) for x in sigma[:3]],
    }
    if e2e:
        out["e2e"] = e2e
        out["e2e_numpy"] = e2e_np
    if rank == 0 and world == 1 and not args.no_cpu and not sparse:
        out["cpu_baseline"] = cpu_baseline(A, cfgd, cfg, Pi, args, df, mode)
    if rank == 0 and world == 1 and not args.no_cpu and sparse:
        out["cpu_baseline"] = cpu_baseline_sparse(indptr, colv, valv, cfgd, cfg, Pi, args, df)
    if rank == 0 and world == 1 and not sparse and not args.no_spmm:
        out["spmm_c3"] = spmm_probe(dev)
    if rank == 0 and world == 1 and args.config == "c2" and not args.no_c4gemm:
        out["gemm_c4"] = gemm_c4_probe(dev, bf16)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def count_launches(step):
    """Count our kernels launched by one step using the CUDA profiler API is
    not available here; instead count C-ABI kernel-launching calls."""
    from paper_1504_05477_b200 import _lib

    L = _lib.load()
    counted = {"n": 0}
    orig = {}
    for name in _lib.exported_symbols():
        if name in ("rsvd_last_error", "rsvd_abi_version", "rsvd_sm_count", "rsvd_gauss_fill") or name.endswith("_ws_bytes"):
            continue
        fn = getattr(L, name)
        orig[name] = fn

        def wrap(*a, _fn=fn, _name=name):
            counted["n"] += LAUNCHES_PER_CALL.get(_name, 1)
            return _fn(*a)

        setattr(L, name, wrap)
    try:
        step()
    finally:
        for name, fn in orig.items():
            setattr(L, name, fn)
    return counted["n"]


# kernels launched per C-ABI call (see csrc/*.cu)
LAUNCHES_PER_CALL = {"rsvd_gemm_tn": 2, "rsvd_colreduce": 2, "rsvd_canonicalize_signs": 3, "rsvd_jacobi_sweeps": 5,
                     "rsvd_eig_select": 2, "rsvd_col_absargmax": 2}


def cpu_baseline(A_dev, cfgd, cfg, Pi, args, df=None, mode="exact"):
    """The reference algorithm (oracle port) on the box's host cores, one
    full factorization; with the device result `df` also the north_star
    parity of this run: max relative error of all k singular values, of the
    per-vector captured variance ||A^T z_i||^2 (metrics.py:136) and of the
    spectral error ||A - Z Z^T A||_2 (the reference's restarted power
    estimator, metrics.py:102-122 / factor.py:217-261, run on the GPU for both
    Z's with identical starts and stopping rule), all on the same A."""
    res, r = reference_sample(A_dev.cpu().numpy(), cfgd, cfg, Pi, budget_s=args.cpu_budget, return_result=True)
    if df is not None:
        import torch

        sig = df.sigma.double().cpu().numpy()
        A64 = A_dev.double()
        if cfgd.get("pca"):
            A64 -= A64.mean(0, keepdim=True)
        cap = (A64.T @ df.Z.double()).pow(2).sum(0).cpu().numpy()
        Zref = torch.from_numpy(np.ascontiguousarray(r.Z)).to(A64.device)
        cap_ref = (A64.T @ Zref).pow(2).sum(0).cpu().numpy()
        del A64
        tol = 1e-10 if A_dev.dtype == torch.float64 else 1e-4
        res["parity"] = {"sigma_rel_max": float(np.max(np.abs(sig - r.sigma) / r.sigma)),
                         "sigma_rel_median": float(np.median(np.abs(sig - r.sigma) / r.sigma)),
                         "captured_variance_rel_max": float(np.max(np.abs(cap - cap_ref) / cap_ref)),
                         "tolerance": tol, "replaced_columns_reference": len(r.replaced),
                         "replaced_columns_ours": (int(df.deflated.sum()) if df.deflated is not None else None)}
        if not args.no_spectral:
            res["parity"]["spectral_error"] = spectral_parity(A_dev, cfgd, df.Z, r.Z, args.spectral_iters)
        res["parity"]["pass"] = bool(res["parity"]["sigma_rel_max"] <= tol and
                                     res["parity"]["captured_variance_rel_max"] <= tol and
                                     res["parity"].get("spectral_error", {}).get("rel", 0.0) <= max(tol, 1e-6))
        if A_dev.dtype == torch.float32 and not args.no_fp64:
            res["parity_fp64_mode"] = mode_leg(A_dev, cfgd, cfg, Pi, r, "fp64")
        if A_dev.dtype == torch.float32 and mode != "fp32" and not args.no_fp32:
            res["parity_fp32_mode"] = mode_leg(A_dev, cfgd, cfg, Pi, r, "fp32")
    return res


def _csr_reference_worker(path, out_path, k, q, p, seed):
    """Child process of cpu_baseline_sparse: the oracle on the host CSR."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import rsvd_oracle as o

    z = np.load(path)
    op = o.CsrOp(int(z["rows"]), int(z["cols"]), z["indptr"], z["col"], z["val"])
    t0 = time.perf_counter()
    r = o.factorize(op, k, "bk", q=q, p=p, seed=seed)
    np.savez(out_path, sigma=r.sigma, Z=r.Z, secs=time.perf_counter() - t0, replaced=len(r.replaced))


def cpu_baseline_sparse(indptr, colv, valv, cfgd, cfg, Pi, args, df):
    """C3's host reference: the oracle's CsrOp (int64 indices, float64 values,
    matrix.py:117-119; its SpMM kernels _kernels.pyx:74-113, OpenMP-sliced but
    bitwise identical) on the same matrix and Pi, in a child process with a
    wall-clock budget (--cpu-budget-sparse). Most of its time is the
    reference's per-column _mgs of the 200000 x 1600 basis (BLAS-2, ~8 TB of
    memory traffic) and its cyclic Jacobi at w = 1600. When it does not finish
    the run is reported as DNF rather than extrapolated; when it finishes the
    parity block is the dense configs': sigma, per-vector captured variance
    ||A^T z_i||^2 (metrics.py:136) and the spectral error ||A - Z Z^T A||_2
    (restarted estimator, metrics.py:102-122), all through an FP64 copy of the
    CSR on the device, plus this path's fp64 mode on the same A and Pi."""
    import multiprocessing as mp
    import tempfile

    import torch

    budget = args.cpu_budget_sparse
    n, d = cfgd["n"], cfgd["d"]
    tmp = tempfile.mkdtemp(prefix="rsvd_c3_")
    path, out_path = os.path.join(tmp, "csr.npz"), os.path.join(tmp, "ref.npz")
    np.savez(path, rows=n, cols=d, indptr=indptr.cpu().numpy().astype(np.int64),
             col=colv.cpu().numpy().astype(np.int64), val=valv.cpu().numpy().astype(np.float64))
    ctx = mp.get_context("spawn")
    proc = ctx.Process(target=_csr_reference_worker, args=(path, out_path, cfg.k, cfg.q, cfg.p, cfg.seed))
    t0 = time.perf_counter()
    proc.start()
    proc.join(budget)
    elapsed = time.perf_counter() - t0
    res = {"unit": "ms", "cores": os.cpu_count() or 1, "kind": "port", "budget_s": budget,
           "sample": ("one full factorization by the reference algorithm (oracle port: its CSR SpMM kernels, "
                      "per-column CGS2 _mgs, C Jacobi) on the same CSR (int64 / float64) and Pi, in a child process "
                      f"with a {budget:.0f} s wall-clock budget")}
    if proc.is_alive():
        proc.terminate()
        proc.join()
        res.update({"value": None, "dnf": True, "elapsed_s": elapsed,
                    "reason": "did not finish within the budget: the reference's per-column _mgs of the "
                              f"{n} x {cfg.p * (cfg.resolve_q(d) + 1)} basis is BLAS-2 (TB of memory traffic) and "
                              "its Jacobi runs at w = 1600; not extrapolated"})
        return res
    r = np.load(out_path)
    res.update({"value": float(r["secs"]) * 1e3, "dnf": False})
    from paper_1504_05477_b200 import metrics as M
    from paper_1504_05477_b200.operators import CsrDeviceOp

    op64 = CsrDeviceOp(indptr, colv, valv.double(), d)
    z_ref = r["Z"]
    sig_ref = r["sigma"]
    cap_ref = M.captured_variance(op64, z_ref)
    res["reference_output"] = {"sigma": [float(x) for x in sig_ref],
                               "captured_variance": [float(x) for x in cap_ref]}

    def block(sig, Z, replaced):
        cap = M.captured_variance(op64, Z)
        out = {"sigma_rel_max": float(np.max(np.abs(sig - sig_ref) / sig_ref)),
               "sigma_rel_median": float(np.median(np.abs(sig - sig_ref) / sig_ref)),
               "captured_variance_rel_max": float(np.max(np.abs(cap - cap_ref) / cap_ref)),
               "tolerance": 1e-4, "replaced_columns_reference": int(r["replaced"]),
               "replaced_columns_ours": replaced}
        return out

    res["parity"] = block(df.sigma.double().cpu().numpy(), df.Z,
                          int(df.deflated.sum()) if df.deflated is not None else None)
    if not args.no_spectral:
        t1 = time.perf_counter()
        sp = {}
        for name, Z in (("ours", df.Z), ("reference_Z", np.ascontiguousarray(z_ref))):
            best, its = M.spectral_norm_batched(M._Deflated(op64, M._as_device_z(Z, op64)),
                                                max_iters=args.spectral_iters)
            sp[name] = float(np.max(best))
            sp[name + "_iterations"] = [int(x) for x in its]
        sp["rel"] = abs(sp["ours"] - sp["reference_Z"]) / sp["reference_Z"]
        sp["max_iters"] = args.spectral_iters
        sp["seconds"] = time.perf_counter() - t1
        res["parity"]["spectral_error"] = sp
    pa = res["parity"]
    pa["pass"] = bool(pa["sigma_rel_max"] <= 1e-4 and pa["captured_variance_rel_max"] <= 1e-4 and
                      pa.get("spectral_error", {}).get("rel", 0.0) <= 1e-4)
    if not args.no_fp64:
        from paper_1504_05477_b200 import rsvd

        g = rsvd.GraphedFactorization(op64, cfg)
        g.run(Pi)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d64 = g.run(Pi)
        e1.record()
        torch.cuda.synchronize()
        leg = block(d64.sigma.double().cpu().numpy(), d64.Z,
                    int(d64.deflated.sum()) if d64.deflated is not None else None)
        leg.update({"ms": e0.elapsed_time(e1), "dtype": "f64 (CSR FP64 SpMM, f64 small algebra)"})
        res["parity_fp64_mode"] = leg
        del g, d64
    del op64
    torch.cuda.empty_cache()
    return res


def spectral_parity(A_dev, cfgd, Z_ours, Z_ref, max_iters):
    """||A - Z Z^T A||_2 by the reference's estimator (seeds 101/202/303, tol
    1e-9, at most `max_iters` power iterations per start, batched as 3
    columns; metrics.py:36-38, 116-121) for our Z and the reference's Z on
    the same operator (FP64-accurate products of the FP32 A)."""
    import torch

    from paper_1504_05477_b200 import metrics as M
    from paper_1504_05477_b200.operators import DenseDeviceOp

    if cfgd.get("pca"):
        A = A_dev.double()
        A -= A.mean(0, keepdim=True)
        op = DenseDeviceOp(A)
    else:
        op = DenseDeviceOp(A_dev, exact=A_dev.dtype == torch.float32)
    op.prepare()
    t0 = time.perf_counter()
    out = {}
    for name, Z in (("ours", Z_ours), ("reference_Z", np.ascontiguousarray(Z_ref))):
        best, its = M.spectral_norm_batched(M._Deflated(op, M._as_device_z(Z, op)), max_iters=max_iters)
        out[name] = float(np.max(best))
        out[name + "_iterations"] = [int(x) for x in its]
    out["rel"] = abs(out["ours"] - out["reference_Z"]) / out["reference_Z"]
    out["max_iters"] = max_iters
    out["seconds"] = time.perf_counter() - t0
    del op
    torch.cuda.empty_cache()
    return out


def mode_leg(A_dev, cfgd, cfg, Pi, r, mode):
    """Another precision mode of this path on the same A and Pi (graph
    replay, one timed step) and its parity against the same reference run:
    "fp64" = A upcast on the device (as the reference upcasts FP32 input,
    matrix.py:80), FP64 DMMA products; "fp32" = 3xTF32 products with the
    projected basis (fastest; FP32-accurate)."""
    import torch

    from paper_1504_05477_b200 import rsvd
    from paper_1504_05477_b200.operators import DenseDeviceOp

    Aw = A_dev.double() if mode == "fp64" else A_dev
    op = DenseDeviceOp(Aw, center=bool(cfgd.get("pca")))
    g = rsvd.GraphedFactorization(op, cfg)
    g.run(Pi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    df = g.run(Pi)
    e1.record()
    torch.cuda.synchronize()
    sig = df.sigma.cpu().numpy()
    A64 = A_dev.double()
    if cfgd.get("pca"):
        A64 -= A64.mean(0, keepdim=True)
    cap = (A64.T @ df.Z.double()).pow(2).sum(0).cpu().numpy()
    cap_ref = (A64.T @ torch.from_numpy(np.ascontiguousarray(r.Z)).to(A64.device)).pow(2).sum(0).cpu().numpy()
    del A64, op, g, Aw
    torch.cuda.empty_cache()
    return {"ms": e0.elapsed_time(e1), "sigma_rel_max": float(np.max(np.abs(sig - r.sigma) / r.sigma)),
            "captured_variance_rel_max": float(np.max(np.abs(cap - cap_ref) / cap_ref)),
            "tolerance": 1e-4, "dtype": MODE_DTYPE[mode]}


def parity_decomposition(A_dev, cfgd, cfg, Pi, r, sig32, cap32):
    """Where the FP32 path's distance to the reference comes from: the same
    projected (block-Lanczos) construction run in FP64 on the same A and Pi.
    fp32_vs_fp64_same_construction = rounding of the FP32 / 3xTF32 path;
    reference_vs_fp64_projected = the reference's own FP64 power-block
    basis (rsvd.py:244-260) against the same Krylov space built without its
    rounding loss."""
    import torch

    from paper_1504_05477_b200 import krylov, rsvd
    from paper_1504_05477_b200.operators import DenseDeviceOp

    A64 = A_dev.double()
    op = DenseDeviceOp(A64, center=bool(cfgd.get("pca")))
    saved = krylov.BK_BASIS
    krylov.BK_BASIS = "projected"
    try:
        df = rsvd.run_device(op, cfg, Pi=torch.from_numpy(np.ascontiguousarray(Pi)).to(A64.device))
        torch.cuda.synchronize()
    finally:
        krylov.BK_BASIS = saved
    sig = df.sigma.double().cpu().numpy()
    if cfgd.get("pca"):
        A64 -= A64.mean(0, keepdim=True)
    cap = (A64.T @ df.Z.double()).pow(2).sum(0).cpu().numpy()
    del A64, op, df
    torch.cuda.empty_cache()

    def rel(a, b):
        return float(np.max(np.abs(a - b) / np.abs(b)))

    return {"fp32_vs_fp64_same_construction": {"sigma_rel_max": rel(sig32, sig), "captured_variance_rel_max": rel(cap32, cap)},
            "reference_vs_fp64_projected": {"sigma_rel_max": rel(r.sigma, sig)},
            "note": "FP64 run of this path's projected construction on the same A and Pi"}


def reference_sample(A32, cfgd, cfg, Pi, budget_s=25.0, return_result=False):
    """One full factorization by the reference algorithm on the box's host
    cores: the oracle port (oracle/rsvd_oracle.py) — numpy/OpenBLAS products
    as the reference's python backend (_kernels_py.py:48-49), the C
    restatement of its compiled Jacobi (_kernels.pyx:127-192), its per-column
    _mgs — on the same A upcast to FP64 (matrix.py:80) and the same Pi.
    Timed like PartialSvdResult.wall_time_ms (rsvd.py:271-282)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import rsvd_oracle as o

    cores = os.cpu_count() or 1
    A = np.ascontiguousarray(A32, dtype=np.float64)
    if cfgd.get("pca"):  # no reference function: the reference on explicitly centered A
        A -= A.mean(axis=0, keepdims=True)
    op = o.DenseOp(A)
    op.apply(Pi[:, :1])  # BLAS thread-pool warm-up outside the timer
    variant = cfg.variant.value if hasattr(cfg.variant, "value") else str(cfg.variant)  # RsvdConfig / RefConfig
    t0 = time.perf_counter()
    r = o.factorize(op, cfg.k, variant, q=cfg.q, p=cfg.p, seed=cfg.seed)
    secs = time.perf_counter() - t0
    out = {"value": secs * 1e3, "unit": "ms", "cores": cores, "kind": "port",
            "sample": ("one full factorization of the same workload by the reference algorithm (oracle port: "
                       "numpy/OpenBLAS products like the reference's python backend, C restatement of its "
                       "Jacobi, per-column CGS2 _mgs) on the same A upcast to FP64 and the same Pi; "
                       f"{cores} host threads (OPENBLAS_NUM_THREADS)"),
            "sigma_head": [float(x) for x in r.sigma[:3]]}
    return (out, r) if return_result else out


class RefConfig:
    """RsvdConfig-equivalent scalars for the reference arm, from the oracle's
    restatement of the reference's q resolution (rsvd.py:151-162) -- the
    reference arm imports nothing from the product package."""

    def __init__(self, k, variant, q, seed=0):
        self.k, self.p, self.q, self.seed, self.variant = int(k), int(k), int(q), int(seed), str(variant)

    def resolve_q(self, d):
        return _oracle().resolve_q(self.variant, self.q, d)


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import rsvd_oracle

    return rsvd_oracle


def make_matrix_host(cfgd, seed=1234):
    """The dense configs' construction on the host with numpy only (the
    reference arm runs no GPU code): Haar V from the QR of a seeded d x d
    Gaussian (sign-fixed by diag R), Haar U from the CholeskyQR of a seeded
    n x d Gaussian generated in row chunks (cond(G) ~ 2.6 at C2, exactly
    orthonormal to FP64 rounding), A = U diag(s) V^T (+ noise), FP32. Same
    spectrum / shape / distribution as make_matrix (a different draw: the
    parity legs run on the device-built A inside the measured arm)."""
    import scipy.linalg as sla

    n, d = cfgd["n"], cfgd["d"]
    if cfgd.get("pca"):
        rng = np.random.default_rng(seed)
        W, R = np.linalg.qr(rng.standard_normal((d, d)))
        W *= np.sign(np.diag(R))[None, :]
        lam = np.exp(-np.arange(1, d + 1) / 50.0)
        mu = rng.uniform(-5.0, 5.0, d)
        M = (W * np.sqrt(lam)[None, :]).T.copy()
        A = np.empty((n, d), dtype=np.float32)
        for c, r0 in enumerate(range(0, n, 65536)):
            r1 = min(n, r0 + 65536)
            G = np.random.default_rng([seed, 1, c]).standard_normal((r1 - r0, d))
            A[r0:r1] = G @ M + mu[None, :]
        return A
    rng = np.random.default_rng(seed)
    V, R = np.linalg.qr(rng.standard_normal((d, d)))
    V *= np.sign(np.diag(R))[None, :]
    s = _spectrum(cfgd["spectrum"], d)
    Wt = (V * s[None, :]).T.copy()  # diag(s) V^T
    chunk = 65536
    starts = list(range(0, n, chunk))

    def gauss(c, rows):
        return np.random.default_rng([seed, 2, c]).standard_normal((rows, d))

    S = np.zeros((d, d))
    for c, r0 in enumerate(starts):
        G = gauss(c, min(n, r0 + chunk) - r0)
        S += G.T @ G
    Rc = np.linalg.cholesky(S).T  # S = R^T R, R upper with positive diagonal
    A = np.empty((n, d), dtype=np.float32)
    for c, r0 in enumerate(starts):
        r1 = min(n, r0 + chunk)
        U = sla.solve_triangular(Rc, gauss(c, r1 - r0).T, trans="T", lower=False).T  # G R^-1
        blk = U @ Wt
        if cfgd["noise"]:
            blk += cfgd["noise"] * np.random.default_rng([seed, 3, c]).standard_normal(blk.shape)
        A[r0:r1] = blk
    return A


def run_reference(args):
    """The reference arm: the oracle port of the reference algorithm on the
    host cores, A generated on the host (numpy), Pi from the oracle's bitwise
    restatement of the reference's SeededRng. No CUDA, no product code."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    o = _oracle()
    cfgd = CONFIGS[args.config]
    cfg = RefConfig(cfgd["k"], cfgd["variant"], cfgd["q"], seed=0)
    if cfgd.get("sparse"):
        print(json.dumps({"impl": "reference", "unavailable": "sparse configs: the reference arm is wired for dense "
                          "configs only (C1/C2/C4/C5); C3's CPU baseline runs inside the measured arm"}), flush=True)
        return
    t0 = time.perf_counter()
    A_host = make_matrix_host(cfgd)
    gen_s = time.perf_counter() - t0
    Pi = o.gaussian(cfgd["d"], cfg.p, o.SeededRng(cfg.seed))
    vals = []
    # CPU runs have no warm-up state beyond the BLAS pool (primed inside
    # reference_sample); warm-up steps are still executed, at most 1 of them
    for i in range(min(args.warmup, 1) + args.steps):
        r = reference_sample(A_host, cfgd, cfg, Pi, budget_s=args.cpu_budget)
        if i >= min(args.warmup, 1):
            vals.append(r["value"])
    v = float(np.mean(vals))
    out = {"impl": "reference", "metric": "rank-k block-Krylov SVD wall time", "value": v, "unit": "ms",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v,
           "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": workload_config(args.config, cfgd, cfg, world),
           "cpu_baseline": {"value": v, "unit": "ms", "cores": r["cores"], "kind": r["kind"], "sample": r["sample"]},
           "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "input_generation_s": gen_s,
           "note": "A generated on the host with numpy (same construction and spectrum as the measured arm, "
                   "different draw); no CUDA and no product code on this path"}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip the FP64 parity-mode leg on FP32 configs")
    ap.add_argument("--no-fp32", action="store_true", help="skip the 3xTF32 fp32-mode leg on FP32 configs")
    ap.add_argument("--no-spectral", action="store_true", help="skip the spectral-error parity")
    ap.add_argument("--spectral-iters", type=int, default=20000,
                    help="power iterations per start of the spectral-error estimator (reference: 20000)")
    ap.add_argument("--precision", default=None, choices=["exact", "fp32", "fp64"],
                    help="override the config's precision mode")
    ap.add_argument("--no-c4gemm", action="store_true", help="skip the tensor-bound C4 chain-GEMM leg of the C2 line")
    ap.add_argument("--no-spmm", action="store_true", help="skip the C3 SpMM measurement on dense configs")
    ap.add_argument("--count-launches", action="store_true", default=True)
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    ap.add_argument("--cpu-budget-sparse", type=float, default=1800.0,
                    help="wall-clock budget (s) of C3's host reference run before it is reported as DNF")
    ap.add_argument("--graph", type=int, default=1, help="replay the factorization as a CUDA graph")
    ap.add_argument("--profile-step", action="store_true",
                    help="bracket one eager factorization with cudaProfilerStart/Stop (for ncu "
                         "--profile-from-start off) after the warm-up, then exit")
    args = ap.parse_args()
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None:
        # one process per GPU: relaunch under torch.distributed.run (the driver
        # launches the N > 1 runs this way itself)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout to the one JSON line
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd, env=env))
    if world_env is not None and int(world_env) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    if world_env is not None and int(world_env) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
