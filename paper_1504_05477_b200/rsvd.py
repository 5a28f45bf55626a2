"""Public algorithm API — drop-in for rsvdkit's rsvd module (rsvd.py:1-314).

Same names, signatures, validation order, exceptions and result type as the
reference: ``Variant``, ``RsvdConfig`` (with the block-Krylov odd-q bump,
rsvd.py:157-158), ``derive_q`` / ``derive_q_gap``, ``PartialSvdResult`` (its
``||Z^T Z - I||_max <= 1e-10`` check, rsvd.py:182-185), ``post_process``,
``simultaneous_iteration``, ``block_krylov``, ``sketch_and_solve`` and
``factorize``. The start block Pi is drawn on the host from
``SeededRng(cfg.seed)`` exactly as the reference does (rsvd.py:225, 233);
everything after that runs on the GPU (krylov.py).

Extra keyword arguments (outside RsvdConfig, so reference configs validate
unchanged):
  precision  "auto" (default): float32 input -> "exact", anything else ->
             "fp64" -- the reference's float64 arithmetic (matrix.py:80).
             "exact": A stays FP32 in HBM, Krylov blocks and small algebra
             are FP64 and both products A X / A^T Y are FP64-accurate int8
             tensor-core GEMMs (Ozaki digit planes, csrc/gemm_oz.cu); the
             reference's construction and deflation decisions are kept.
             "fp64": A upcast to FP64 on the device, FP64 DMMA products.
             "fp32": 3xTF32 tensor-core products, FP32 blocks with the
             projected (block-Lanczos) basis, FP64 small algebra, FP64
             re-orthonormalized Z -- fastest, FP32-accurate (opt-in).
  center     implicit mean-centering (PCA): factorizes A - 1 mu^T without
             forming it.
  device     CUDA device for host inputs (default: current device).
  comm       krylov.TorchComm for a row-sharded A (each rank passes its
             rows; results are returned on every rank).
"""

from __future__ import annotations

import enum
import math
import os
import time
import warnings
from dataclasses import dataclass, field

from collections import OrderedDict

import numpy as np
import torch

from . import device as ops
from . import krylov
from .errors import ConvergenceError
from .matrix import DenseMatrix, MatrixOperator, SeededRng, SparseMatrixCSR, as_dense_array, gaussian
from .operators import CsrDeviceOp, DenseDeviceOp

__all__ = [
    "Variant",
    "RsvdConfig",
    "PartialSvdResult",
    "derive_q",
    "derive_q_gap",
    "post_process",
    "simultaneous_iteration",
    "block_krylov",
    "sketch_and_solve",
    "factorize",
]


class Variant(str, enum.Enum):
    SIMULTANEOUS_ITERATION = "si"
    BLOCK_KRYLOV = "bk"
    SKETCH = "sketch"


def _variant(v):
    return v if isinstance(v, Variant) else Variant(str(v).lower())


def _odd(q):
    return q + 1 - (q % 2)  # rsvd.py:52-53


def _check_common(d, epsilon, C):
    if d < 2:
        raise ValueError("d must be at least 2")
    if not 0 < epsilon < 1:
        raise ValueError("epsilon must be in (0, 1)")
    if not C > 0:
        raise ValueError("C must be positive")


def derive_q(variant, d, epsilon, C=4.0):
    """rsvd.py:56-75 — SI: ceil(C ln d / eps); BK: ceil(C ln d / sqrt(eps)), odd."""
    variant = _variant(variant)
    if variant is Variant.SKETCH:
        return 0
    _check_common(d, epsilon, C)
    if variant is Variant.SIMULTANEOUS_ITERATION:
        return math.ceil(C * math.log(d) / epsilon)
    return _odd(math.ceil(C * math.log(d) / math.sqrt(epsilon)))


def derive_q_gap(variant, d, epsilon, gap, C=4.0):
    """rsvd.py:78-100 — gap-aware count, gap clamped to 1."""
    variant = _variant(variant)
    if variant is Variant.SKETCH:
        return 0
    if d < 2:
        raise ValueError("d must be at least 2")
    if not 0 < epsilon < 1:
        raise ValueError("epsilon must be in (0, 1)")
    if not gap > 0:
        raise ValueError("gap must be positive")
    if not C > 0:
        raise ValueError("C must be positive")
    g = min(1.0, float(gap))
    base = C * math.log(d / epsilon)
    if variant is Variant.SIMULTANEOUS_ITERATION:
        return math.ceil(base / g)
    return _odd(math.ceil(base / math.sqrt(g)))


@dataclass(frozen=True)
class RsvdConfig:
    """rsvd.py:103-162 — factorization request (exactly one of q / epsilon;
    gap needs epsilon; p defaults to k and must be >= k)."""

    k: int
    variant: Variant
    p: int | None = None
    q: int | None = None
    epsilon: float | None = None
    gap: float | None = None
    C: float = 4.0
    seed: int = 0
    reorthonormalize_every: int = 1

    def __post_init__(self):
        object.__setattr__(self, "variant", _variant(self.variant))
        if self.k < 1:
            raise ValueError("k must be at least 1")
        p = self.k if self.p is None else int(self.p)
        if p < self.k:
            raise ValueError("block width p must be at least k")
        object.__setattr__(self, "p", p)
        if self.variant is not Variant.SKETCH and (self.q is None) == (self.epsilon is None):
            raise ValueError("give exactly one of q or epsilon")
        if self.q is not None and self.q < 0:
            raise ValueError("q must be nonnegative")
        if self.epsilon is not None and not 0 < self.epsilon < 1:
            raise ValueError("epsilon must be in (0, 1)")
        if self.gap is not None:
            if self.epsilon is None:
                raise ValueError("gap requires epsilon")
            if not self.gap > 0:
                raise ValueError("gap must be positive")
        if not self.C > 0:
            raise ValueError("C must be positive")
        if not 0 <= int(self.seed) < (1 << 64):
            raise ValueError("seed must fit in an unsigned 64-bit integer")
        if self.reorthonormalize_every < 0:
            raise ValueError("reorthonormalize_every must be nonnegative")

    def resolve_q(self, d):
        """rsvd.py:151-162 — BK bumps an explicit even q >= 1 to odd."""
        if self.variant is Variant.SKETCH:
            return 0
        if self.q is not None:
            q = int(self.q)
            return _odd(q) if (self.variant is Variant.BLOCK_KRYLOV and q >= 1) else q
        if self.gap is not None:
            return derive_q_gap(self.variant, d, self.epsilon, self.gap, self.C)
        return derive_q(self.variant, d, self.epsilon, self.C)


def _wrap_dense(arr, finite_checked=False):
    """DenseMatrix around a freshly produced float64 array without a second copy."""
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    if not finite_checked and not np.all(np.isfinite(arr)):
        raise ValueError("dense matrix entries must be finite")
    arr.setflags(write=False)
    obj = object.__new__(DenseMatrix)
    object.__setattr__(obj, "data", arr)
    return obj


@dataclass(frozen=True)
class PartialSvdResult:
    """rsvd.py:165-189 — orthonormal Z (n x k), approximate singular values
    (descending, >= 0), diagnostics. The orthonormality check uses the
    device-computed ||Z^T Z - I||_max when the factorization produced it."""

    Z: DenseMatrix
    approx_singular_values: np.ndarray
    q_used: int
    wall_time_ms: float
    variant: Variant
    seed: int
    _z_ortho_err: float | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        sv = np.array(self.approx_singular_values, dtype=np.float64, copy=True)
        if sv.ndim != 1 or np.any(sv < 0) or np.any(np.diff(sv) > 0):
            raise ValueError("approximate singular values must be nonnegative descending")
        sv.setflags(write=False)
        object.__setattr__(self, "approx_singular_values", sv)
        err = self._z_ortho_err
        if err is None:
            z = self.Z.data
            err = float(np.max(np.abs(z.T @ z - np.eye(z.shape[1])))) if z.size else 0.0
        if not err <= 1e-10:
            raise ValueError("Z must have orthonormal columns")

    @property
    def k(self):
        return self.Z.cols


# --------------------------------------------------------------------------
# input handling


def _resolve_device(device):
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1504_05477_b200 requires a CUDA device (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


PRECISIONS = ("auto", "exact", "fp64", "fp32")


def _mode(src_dtype, precision):
    """Resolved arithmetic mode: "exact" (FP32 A, FP64-accurate products),
    "fp64" or "fp32". "exact" only differs from "fp64" for FP32 input."""
    if precision not in PRECISIONS:
        raise ValueError("precision must be 'auto', 'exact', 'fp64' or 'fp32'")
    f32 = src_dtype in (np.float32, torch.float32)
    if precision in ("auto", "exact"):
        return "exact" if f32 else "fp64"
    return precision


def _work_dtype(src_dtype, precision):
    """dtype A is stored in on the device."""
    return torch.float64 if _mode(src_dtype, precision) == "fp64" else torch.float32


def make_operator(A, precision="auto", center=False, device=None, comm=None, n_total=None, row_offset=0):
    """Upload / wrap A as a device operator (the as_operator step,
    matrix.py:260-263). Dense host input is validated like DenseMatrix."""
    if isinstance(A, (DenseDeviceOp, CsrDeviceOp)):
        return A
    if isinstance(A, MatrixOperator):  # the reference's as_operator(A) handle: its host matrix
        A = A.matrix
    if isinstance(A, SparseMatrixCSR):
        if center:
            raise ValueError("implicit centering is supported for dense A only")
        dev = _resolve_device(device)
        dt = _work_dtype(np.float64, precision)
        idx = torch.int64 if A.nnz >= 2**31 - 1 else torch.int32
        indptr = torch.from_numpy(A.row_ptr.astype(np.int64)).to(device=dev, dtype=idx)
        col = torch.from_numpy(A.col_idx).to(device=dev, dtype=idx)
        val = torch.from_numpy(A.values).to(device=dev, dtype=dt)
        return CsrDeviceOp(indptr, col, val, A.cols, n_total=n_total, row_offset=row_offset)
    if isinstance(A, torch.Tensor):
        dev = A.device if A.is_cuda else _resolve_device(device)
        dt = _work_dtype(A.dtype, precision)
        exact = _mode(A.dtype, precision) == "exact"
        if A.dim() != 2:
            raise ValueError("dense matrix data must be 2-D")
        if A.is_cuda:
            t = A.to(device=dev, dtype=dt)
        else:
            # host input: DMA straight into a preallocated device tensor
            # (55 GB/s from pinned memory on PCIe Gen5 x16, vs 24 GB/s measured
            # for .to(cuda) of the same pinned tensor); cast on the device
            src = A if A.is_contiguous() else A.contiguous()
            raw = torch.empty(src.shape, dtype=src.dtype, device=dev)
            raw.copy_(src, non_blocking=src.is_pinned())
            t = raw if raw.dtype == dt else raw.to(dt)
        if not bool(torch.isfinite(t).all()):
            raise ValueError("dense matrix entries must be finite")
        return DenseDeviceOp(t.contiguous(), n_total=n_total, row_offset=row_offset, center=center, comm=comm,
                             exact=exact)
    src_dtype = np.asarray(A).dtype if not isinstance(A, DenseMatrix) else np.float64
    arr = as_dense_array(A) if not (isinstance(A, np.ndarray) and A.dtype == np.float32) else np.asarray(A)
    if arr.ndim != 2:
        raise ValueError("dense matrix data must be 2-D")
    if not np.all(np.isfinite(arr)):
        raise ValueError("dense matrix entries must be finite")
    dev = _resolve_device(device)
    dt = _work_dtype(src_dtype, precision)
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(device=dev, dtype=dt, non_blocking=False)
    return DenseDeviceOp(t, n_total=n_total, row_offset=row_offset, center=center, comm=comm,
                         exact=_mode(src_dtype, precision) == "exact")


# --------------------------------------------------------------------------
# device pipeline


@dataclass
class DeviceFactorization:
    """Device-resident outcome of one factorization (no host copies)."""

    Z: torch.Tensor  # n_local x k FP64
    sigma: torch.Tensor  # k FP64
    info: torch.Tensor  # Jacobi [converged, sweeps, ...]
    off: torch.Tensor
    zerr: torch.Tensor
    q_used: int
    deflated: torch.Tensor | None = None


def _sign_fn_for(comm):
    if comm is None or getattr(comm, "world", 1) == 1:
        return None
    from .dist import sharded_canonicalize_signs

    return lambda Z: sharded_canonicalize_signs(Z, comm)


def run_device(op, cfg, comm=None, Pi=None):
    """The whole path on the device for an already-uploaded operator.
    Validation as _run (rsvd.py:263-270); no host synchronisation. ``Pi`` is
    the host start block (default: drawn from SeededRng(cfg.seed)) or an
    already-uploaded device tensor."""
    n, d = op.shape
    if cfg.k > min(n, d):
        raise ValueError("k must not exceed min(n, d)")
    q = cfg.resolve_q(d)
    c = comm if comm is not None else krylov.LocalComm()
    n_total, row_offset = op.n_total, op.row_offset
    p = cfg.p
    if cfg.variant is Variant.BLOCK_KRYLOV and p > n:
        raise ValueError("block width p exceeds n; no Krylov block fits")
    if Pi is None:
        Pi = gaussian(d, p, SeededRng(cfg.seed)).data
    if isinstance(Pi, torch.Tensor) and Pi.is_cuda:
        pi_dev = Pi
    else:
        pi_dev = torch.from_numpy(np.array(Pi, copy=True)).to(device=op.device, dtype=op.dtype, non_blocking=True)
    ws = krylov.Workspace(op.device, p)
    op.prepare()  # exact mode: digit planes of A, inside the timed / captured region
    deflated = None
    if cfg.variant is Variant.SIMULTANEOUS_ITERATION:
        Q = krylov.si_basis(ops, c, op, pi_dev, q, cfg.reorthonormalize_every, ws, n_total, row_offset)
        q_used = q
    elif cfg.variant is Variant.BLOCK_KRYLOV:
        br = krylov.bk_basis(ops, c, op, pi_dev, q, ws, n_total, row_offset)
        Q, q_used, deflated, W = br.Q, br.q_used, br.deflated, br.W
    else:
        Q = krylov.sketch_basis(ops, c, op, pi_dev, ws, n_total, row_offset)
        q_used = 0
    rr = krylov.rayleigh_ritz(ops, c, op, Q, cfg.k, n_total, row_offset, sign_fn=_sign_fn_for(comm),
                              W=W if cfg.variant is Variant.BLOCK_KRYLOV else None)
    return DeviceFactorization(rr.Z, rr.sigma, rr.info, rr.off, rr.zerr, q_used, deflated)


class GraphedFactorization:
    """One factorization of a fixed operator/config captured as a CUDA graph.

    Everything run_device enqueues is stream-ordered and free of host
    synchronisation (data-dependent steps are device-side predicates), so the
    ~2000 kernel launches of a factorization replay as one graph launch. The
    start block is copied into a static device buffer before each replay; the
    outputs are static device tensors (valid until the next replay)."""

    def __init__(self, op, cfg, comm=None):
        self.op, self.cfg, self.comm = op, cfg, comm
        d = op.shape[1]
        self.pi = torch.empty((d, cfg.p), dtype=op.dtype, device=op.device)
        self.graph = None
        self.out = None

    def _capture(self):
        # two eager runs size every workspace before capture (no allocation
        # growth may happen while capturing)
        for _ in range(2):
            run_device(self.op, self.cfg, comm=self.comm, Pi=self.pi)
        torch.cuda.synchronize(self.op.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.out = run_device(self.op, self.cfg, comm=self.comm, Pi=self.pi)
        self.graph = g

    def run(self, Pi=None):
        if Pi is None:
            Pi = gaussian(self.op.shape[1], self.cfg.p, SeededRng(self.cfg.seed)).data
        src = Pi if isinstance(Pi, torch.Tensor) else torch.from_numpy(np.array(Pi, copy=True))
        self.pi.copy_(src, non_blocking=True)
        if self.graph is None:
            self._capture()
        self.graph.replay()
        return self.out


def _to_host(Z):
    """D2H of the result through page-locked memory: a DMA at full link
    speed instead of a staged copy into freshly faulted pageable pages. The
    returned array owns its buffer (torch's caching host allocator recycles
    the block once the caller drops the result)."""
    if not Z.is_cuda:
        return Z.numpy()
    h = torch.empty(Z.shape, dtype=Z.dtype, pin_memory=True)
    h.copy_(Z, non_blocking=True)
    torch.cuda.current_stream(Z.device).synchronize()
    return h.numpy()


def _finish(df, cfg, t0, gather_z=None):
    info = df.info.cpu()
    off = float(df.off.cpu()[0])
    if int(info[0]) != 1:
        raise ConvergenceError(
            f"Jacobi did not converge in {krylov.JACOBI_MAX_SWEEPS} sweeps (off-diagonal mass {off:.3e})",
            residual=off,
        )
    Z = df.Z if gather_z is None else gather_z(df.Z)
    finite = False
    if Z.is_cuda and Z.numel():
        # DenseMatrix's finiteness rule (matrix.py:80-85) checked on the device:
        # |z| <= 1 for orthonormal columns, so a column sum is finite iff
        # every entry of the column is
        finite = bool(torch.isfinite(ops.colreduce(Z, square=False)).all())
        if not finite:
            raise ValueError("dense matrix entries must be finite")
    z_host = _to_host(Z)
    sigma = df.sigma.cpu().numpy()
    zerr = float(df.zerr.cpu()[0])
    elapsed_ms = (time.perf_counter() - t0) * 1e3
    return PartialSvdResult(
        Z=_wrap_dense(z_host, finite_checked=finite),
        approx_singular_values=sigma,
        q_used=df.q_used,
        wall_time_ms=elapsed_ms,
        variant=cfg.variant,
        seed=int(cfg.seed),
        _z_ortho_err=zerr,
    )


# Public-API graph cache: a dense single-GPU call re-uses a persistent device
# buffer for A of its shape and replays the factorization as one CUDA graph
# (GraphedFactorization); the ~1000 kernels otherwise pay host launch cost on
# every call. The captured factorization is data-independent (every
# data-dependent step is device-predicated), so the replay is exact for any A
# of the same shape / dtype / config. One entry (LRU); RSVD_GRAPH_CACHE=0
# turns it off.
_GRAPH_CACHE = OrderedDict()
_GRAPH_CACHE_SIZE = 1


def _graph_cache_key(A, cfg, precision, device, center=False):
    if os.environ.get("RSVD_GRAPH_CACHE", "1") != "1":
        return None
    if isinstance(A, torch.Tensor):
        if A.dim() != 2 or A.dtype not in (torch.float32, torch.float64):
            return None
        src = np.float32 if A.dtype == torch.float32 else np.float64
        shape = tuple(A.shape)
        dev = A.device if A.is_cuda else _resolve_device(device)
    elif isinstance(A, DenseMatrix) or (isinstance(A, np.ndarray) and A.ndim == 2 and
                                        A.dtype in (np.float32, np.float64)):
        src = np.float64 if isinstance(A, DenseMatrix) else A.dtype.type
        shape = tuple(A.shape)
        dev = _resolve_device(device)
    else:
        return None
    dt = _work_dtype(src, precision)
    q = cfg.resolve_q(shape[1])
    return (shape, dt, str(dev), cfg.k, cfg.p, q, cfg.variant, int(cfg.seed), cfg.reorthonormalize_every,
            bool(center), _mode(src, precision))


class _PageableUploader:
    """H2D of a pageable host array through two pinned staging buffers: host
    threads copy chunk i + 1 into one buffer while the DMA engine moves chunk
    i out of the other (a plain copy from pageable memory goes through the
    driver's own single-threaded staging: ~14 GB/s measured at C2, 2 GB in
    ~140 ms). Casting to the device dtype happens in the host copy."""

    CHUNK_BYTES = 64 << 20
    THREADS = min(16, os.cpu_count() or 1)

    def __init__(self):
        self.bufs = None
        self.events = None
        self.pool = None

    def _setup(self):
        if self.bufs is None:
            from concurrent.futures import ThreadPoolExecutor

            self.bufs = [torch.empty(self.CHUNK_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
            self.events = [None, None]
            self.pool = ThreadPoolExecutor(max_workers=self.THREADS)

    def upload(self, dst, arr, stream=None, on_chunk=None):
        """``stream``: the stream the DMAs are issued on (default: the current
        one); ``on_chunk(n_elements, event)`` is called after each chunk's DMA
        has been enqueued, with the flat element count uploaded so far and the
        event that marks its arrival."""
        self._setup()
        src = arr.reshape(-1)
        flat = dst.view(-1)
        esize = dst.element_size()
        npdt = np.float32 if dst.dtype == torch.float32 else np.float64
        per = self.CHUNK_BYTES // esize
        stream = stream or torch.cuda.current_stream(dst.device)
        for i, off in enumerate(range(0, src.size, per)):
            m = min(per, src.size - off)
            slot = i % 2
            if self.events[slot] is not None:
                self.events[slot].synchronize()  # the DMA out of this buffer is done
            host = self.bufs[slot][: m * esize].numpy().view(npdt)
            nt = self.THREADS if m >= (1 << 20) else 1
            bounds = [(m * t) // nt for t in range(nt + 1)]

            def cp(t, host=host, off=off, bounds=bounds):
                a, b = bounds[t], bounds[t + 1]
                if b > a:  # numpy releases the GIL for the copy
                    np.copyto(host[a:b], src[off + a: off + b], casting="unsafe")

            list(self.pool.map(cp, range(nt)))
            with torch.cuda.stream(stream):
                flat[off: off + m].copy_(self.bufs[slot][: m * esize].view(dst.dtype), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            self.events[slot] = ev
            if on_chunk is not None:
                on_chunk(off + m, ev)
        for ev in self.events:
            if ev is not None:
                ev.synchronize()


_UPLOADER = _PageableUploader()


_COPY_STREAMS = {}
# rows per panel of the pipelined upload (a multiple of 32)
_PANEL_BYTES = 256 << 20


def _upload_pipelined(buf, A, op):
    """Exact mode, host input: the upload runs on a copy stream in row panels;
    as each panel lands, the caller's stream adds its column sums (the
    finiteness check) and cuts its digit planes (OzPlanes.refresh_rows), so
    that only the last panel's share of that work (C2: ~1.5 ms in all) is left
    when the upload ends. Returns the FP64 column sums (device)."""
    dev = buf.device
    main = torch.cuda.current_stream(dev)
    cs = _COPY_STREAMS.get(dev)
    if cs is None:
        cs = _COPY_STREAMS[dev] = torch.cuda.Stream(device=dev)
    start = torch.cuda.Event()
    start.record(main)
    cs.wait_event(start)  # earlier work on the caller's stream may still read buf
    n, d = buf.shape
    rows = max(32, (_PANEL_BYTES // max(1, d * buf.element_size())) // 32 * 32)
    sums = torch.zeros(d, dtype=torch.float64, device=dev)
    part = torch.empty(d, dtype=torch.float64, device=dev)
    done = [0]

    def rows_landed(r1, ev):
        # rows [done, r1) are in HBM once ev has fired
        r0 = done[0]
        if r1 <= r0:
            return
        main.wait_event(ev)
        ops.colreduce(buf[r0:r1], False, part)
        sums.add_(part)
        op.oz.refresh_rows(buf, r0, r1 - r0)
        done[0] = r1

    if isinstance(A, torch.Tensor):
        src = A if A.is_contiguous() else A.contiguous()
        for r0 in range(0, n, rows):
            r1 = min(n, r0 + rows)
            with torch.cuda.stream(cs):
                buf[r0:r1].copy_(src[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            rows_landed(r1, ev)
    else:
        def on_chunk(n_el, ev):
            full = n_el // d  # complete rows uploaded so far
            r1 = n if full >= n else full // rows * rows
            rows_landed(r1, ev)

        _UPLOADER.upload(buf, A, stream=cs, on_chunk=on_chunk)
    return sums


def _pipelined_ok(A, op, buf):
    """Host input of the buffer's dtype, exact mode, big enough to be worth panels."""
    if getattr(op, "oz", None) is None or not getattr(op, "external_planes", False):
        return False
    if buf.numel() * buf.element_size() < 2 * _PANEL_BYTES:
        return False
    if isinstance(A, torch.Tensor):
        return (not A.is_cuda) and A.is_pinned() and A.dtype == buf.dtype
    return isinstance(A, np.ndarray) and A.dtype == np.float32 and A.flags.c_contiguous


def _upload_into(buf, A, op=None, defer_check=False):
    """Copy host / device A into the persistent buffer (DMA from pinned
    memory), with the dense-input validation of make_operator. With ``op`` in
    exact mode and ``external_planes`` set, the digit planes of A are cut here
    (pipelined with the upload when the input allows it). ``defer_check``:
    return the column sums without the host-side finiteness check (the caller
    checks after launching the factorization)."""
    if op is not None and _pipelined_ok(A, op, buf):
        sums = _upload_pipelined(buf, A, op)
        if not defer_check and not bool(torch.isfinite(sums).all()):
            raise ValueError("dense matrix entries must be finite")
        return sums
    if isinstance(A, torch.Tensor):
        src = A if A.is_contiguous() else A.contiguous()
        if src.dtype == buf.dtype:
            buf.copy_(src, non_blocking=(not src.is_cuda) and src.is_pinned())
        else:
            buf.copy_(src.to(device=buf.device, non_blocking=(not src.is_cuda) and src.is_pinned()))
    else:
        arr = as_dense_array(A) if not (isinstance(A, np.ndarray) and A.dtype == np.float32) else np.asarray(A)
        arr = np.ascontiguousarray(arr)
        if arr.nbytes >= 2 * _PageableUploader.CHUNK_BYTES:
            _UPLOADER.upload(buf, arr)
        else:
            with warnings.catch_warnings():  # read-only source (DenseMatrix data): only read by the copy
                warnings.simplefilter("ignore", UserWarning)
                buf.copy_(torch.from_numpy(arr))
    # one pass, no temporaries: FP64 column sums are finite iff every entry is
    # (an FP32 column cannot overflow an FP64 sum; for FP64 input a sum could
    # only overflow with entries near 1e308)
    sums = torch.empty(buf.shape[1], dtype=torch.float64, device=buf.device)
    ops.colreduce(buf, False, sums)
    if op is not None and getattr(op, "oz", None) is not None and getattr(op, "external_planes", False):
        op.oz.refresh(buf)
    if not defer_check and not bool(torch.isfinite(sums).all()):
        raise ValueError("dense matrix entries must be finite")
    return sums


def _run(A, cfg, expected, precision="auto", center=False, device=None, comm=None):
    if cfg.variant is not expected:
        raise ValueError(f"config variant is {cfg.variant.value}, not {expected.value}")
    key = None
    if comm is None or getattr(comm, "world", 1) == 1:
        key = _graph_cache_key(A, cfg, precision, device, center)
    if key is not None:
        shape, dt, dev = key[0], key[1], torch.device(key[2])
        if shape[0] == 0 or shape[1] == 0 or cfg.k > min(shape):
            key = None  # let the eager path raise the reference's errors
    if key is not None:
        entry = _GRAPH_CACHE.pop(key, None)
        if entry is None:
            while len(_GRAPH_CACHE) >= _GRAPH_CACHE_SIZE:
                _GRAPH_CACHE.popitem(last=False)
            buf = torch.empty(shape, dtype=dt, device=dev)
            if center:
                buf.zero_()
            op = DenseDeviceOp(buf, center=center, exact=key[-1] == "exact")
            # the planes are cut by _upload_into (per row panel, as the upload lands)
            op.external_planes = op.oz is not None
            pi_host = gaussian(shape[1], cfg.p, SeededRng(cfg.seed)).data
            pi_dev = torch.from_numpy(np.array(pi_host, copy=True)).to(device=dev, dtype=op.dtype)
            entry = [buf, op, GraphedFactorization(op, cfg), pi_dev, 0]
        _GRAPH_CACHE[key] = entry
        buf, op, graphed, pi, calls = entry
        entry[4] = calls + 1
        with torch.cuda.device(dev):
            sums = _upload_into(buf, A, op=op, defer_check=True)
            if center:
                op.set_column_sums(sums)
            t0 = time.perf_counter()
            # the first call of a shape runs eagerly; a repeated shape is
            # captured once and replayed from then on
            df = run_device(op, cfg, Pi=pi) if calls == 0 else graphed.run(pi)
            # input validation (matrix.py:80-85) while the factorization runs
            if not bool(torch.isfinite(sums).all()):
                raise ValueError("dense matrix entries must be finite")
            return _finish(df, cfg, t0)
    n_total = row_offset = None
    if comm is not None and getattr(comm, "world", 1) > 1:
        n_total, row_offset = comm.n_total, comm.row_offset
    op = make_operator(A, precision=precision, center=center, device=device, comm=comm,
                       n_total=n_total, row_offset=row_offset or 0)
    dev = op.device
    with torch.cuda.device(dev):
        t0 = time.perf_counter()
        df = run_device(op, cfg, comm=comm)
        gather = None
        if comm is not None and getattr(comm, "world", 1) > 1:
            from .dist import gather_rows

            gather = lambda Z: gather_rows(Z, comm)  # noqa: E731
        return _finish(df, cfg, t0, gather)


def simultaneous_iteration(A, cfg, **kw):
    """rsvd.py:293-295 — randomized simultaneous (power) iteration."""
    return _run(A, cfg, Variant.SIMULTANEOUS_ITERATION, **kw)


def block_krylov(A, cfg, **kw):
    """rsvd.py:298-300 — randomized block Krylov iteration."""
    return _run(A, cfg, Variant.BLOCK_KRYLOV, **kw)


def sketch_and_solve(A, cfg, **kw):
    """rsvd.py:303-305 — basis of A Pi, then post-processing."""
    return _run(A, cfg, Variant.SKETCH, **kw)


def factorize(A, cfg, **kw):
    """rsvd.py:308-314 — dispatch on cfg.variant."""
    if cfg.variant is Variant.SIMULTANEOUS_ITERATION:
        return simultaneous_iteration(A, cfg, **kw)
    if cfg.variant is Variant.BLOCK_KRYLOV:
        return block_krylov(A, cfg, **kw)
    return sketch_and_solve(A, cfg, **kw)


def post_process(A, Q, k, precision="auto", device=None):
    """rsvd.py:200-221 — best rank-l bases inside span(Q) for every l <= k.
    Returns (DenseMatrix Z, sigma) like the reference."""
    op = make_operator(A, precision=precision, device=device)
    qarr = as_dense_array(Q)
    if qarr.shape[1] < k:
        raise ValueError("Q must have at least k columns")
    with torch.cuda.device(op.device):
        qd = torch.from_numpy(qarr).to(device=op.device, dtype=op.dtype)
        G = ops.gram(qd)
        err = float(ops.ortho_error(G).cpu()[0])
        if not err <= 1e-8:
            raise ValueError("Q must have orthonormal columns")
        rr = krylov.rayleigh_ritz(ops, krylov.LocalComm(), op, qd, int(k), op.n_total, 0)
        info = rr.info.cpu()
        if int(info[0]) != 1:
            off = float(rr.off.cpu()[0])
            raise ConvergenceError("Jacobi did not converge", residual=off)
        return _wrap_dense(rr.Z.cpu().numpy()), rr.sigma.cpu().numpy()
