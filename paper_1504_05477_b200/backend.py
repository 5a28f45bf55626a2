"""Kernel-contract conformance module — the five functions the reference
binds at import (backend.py:39-43), with the reference's numpy-in/numpy-out
signatures, computed by the CUDA kernels. Lets
reference-style kernel tests (test_backends.py, test_matrix.py) run against
the GPU.

    gauss_fill(count, state) -> (float64[count], new_state)      _kernels.pyx:31
    mm(a, b) -> a @ b                                             _kernels.pyx:56
    spmm_nt(nrows, indptr, col, val, b)                           _kernels.pyx:74
    spmm_t(nrows, ncols, indptr, col, val, b)                     _kernels.pyx:95
    jacobi_sweeps(m_, v_, tol, max_sweeps) -> (off, sweeps, conv) _kernels.pyx:127
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as ops


def active_backend():
    return "cuda"


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("CUDA backend requires a GPU")
    return torch.device("cuda", torch.cuda.current_device())


def _to(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=_dev(), dtype=dtype)


def gauss_fill(count, state):
    return ops.gauss_fill_host(int(count), int(state))


def mm(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError("mm: shape mismatch")
    A, B = _to(a), _to(b)
    C = torch.empty((a.shape[0], b.shape[1]), dtype=torch.float64, device=A.device)
    ops.gemm_nn(A, B, C)
    return C.cpu().numpy()


def _csr(indptr, col, val):
    return (_to(np.asarray(indptr, dtype=np.int64), torch.int64), _to(np.asarray(col, dtype=np.int64), torch.int64),
            _to(np.asarray(val, dtype=np.float64)))


def spmm_nt(nrows, indptr, col, val, b):
    b = np.ascontiguousarray(b, dtype=np.float64)
    ip, cp, vp = _csr(indptr, col, val)
    B = _to(b)
    C = torch.empty((int(nrows), b.shape[1]), dtype=torch.float64, device=B.device)
    ops.spmm_csr(ip, cp, vp, b.shape[0], B, C)
    return C.cpu().numpy()


def spmm_t(nrows, ncols, indptr, col, val, b):
    b = np.ascontiguousarray(b, dtype=np.float64)
    ip, cp, vp = _csr(indptr, col, val)
    tp, tc, tv = ops.csr_transpose(ip, cp, vp, int(nrows), int(ncols))
    B = _to(b)
    C = torch.empty((int(ncols), b.shape[1]), dtype=torch.float64, device=B.device)
    ops.spmm_csr(tp, tc, tv, int(nrows), B, C)
    return C.cpu().numpy()


def jacobi_sweeps(m_, v_, tol, max_sweeps):
    """In place on the caller's numpy arrays, like the reference."""
    M, V = _to(m_), _to(v_)
    info, off = ops.jacobi_sweeps(M, V, float(tol), int(max_sweeps))
    m_[...] = M.cpu().numpy()
    v_[...] = V.cpu().numpy()
    info = info.cpu().numpy()
    return float(off.cpu()[0]), int(info[1]), bool(info[0])
