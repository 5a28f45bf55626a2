"""Host-facing entry points of the two small factorizations on the hot path
(reference factor.py): ``qr_orthonormalize`` (factor.py:121-129, the public
face of ``_mgs``, factor.py:79-118) and ``symmetric_eig`` (factor.py:132-166),
with the reference's signatures, validation and error behaviour. Both run on
the GPU through the same kernels the factorization uses -- the blocked
BCGS2 + CholeskyQR orthonormalization with deflation and the seeded fill
stream (krylov.orth_block), and the Jacobi kernel of the kernel contract
(device.jacobi_sweeps); there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as ops
from . import krylov
from .errors import ConvergenceError
from .matrix import DenseMatrix, as_dense_array

# Columns per orthonormalization step: one p <= 64 register Cholesky per block.
QR_BLOCK = 64


@dataclass(frozen=True)
class EigResult:
    """factor.py:44-56 -- eigenvalues descending; column i pairs with value i."""

    eigenvalues: np.ndarray
    eigenvectors: DenseMatrix

    def __post_init__(self):
        vals = np.array(self.eigenvalues, dtype=np.float64, copy=True)
        if vals.ndim != 1 or np.any(np.diff(vals) > 0):
            raise ValueError("eigenvalues must be a descending 1-D array")
        vals.setflags(write=False)
        object.__setattr__(self, "eigenvalues", vals)


def _device(device):
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1504_05477_b200 requires a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)


def qr_orthonormalize(M, device=None):
    """Orthonormal basis with M's column count spanning span(M); numerically
    dependent columns (residual <= 1e-12 x the column's norm) are replaced from
    the seeded fill stream, one stream per call like one ``_mgs`` call. Columns
    are processed in blocks of QR_BLOCK, each against the finished prefix."""
    arr = as_dense_array(M)
    n, m = arr.shape
    if n < m:
        raise ValueError("qr_orthonormalize requires rows >= cols")
    dev = _device(device)
    with torch.cuda.device(dev):
        K = krylov.rows_buffer(n, m, torch.float64, dev)
        K.copy_(torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)))
        pb = max(1, min(QR_BLOCK, m))
        ws = krylov.Workspace(dev, pb)
        comm = krylov.LocalComm()
        tmp = krylov.rows_buffer(n, pb, torch.float64, dev)
        running = torch.zeros(1, dtype=torch.int32, device=dev)
        for j0 in range(0, m, pb):
            pw = min(pb, m - j0)
            cur = K[:, j0: j0 + pw]
            ref2 = None
            if j0:  # norms before the projection against the prefix (the first block's come from its Gram)
                ref2 = ws.ref2[:pw]
                ops.colreduce(cur, True, ref2)
            krylov.orth_block(ops, comm, cur, tmp[:, :pw], ws, Qp=K[:, :j0] if j0 else None, ref2=ref2,
                              running=running, n_total=n, row_offset=0)
        return DenseMatrix(K.cpu().numpy())


def symmetric_eig(M, tol=None, max_sweeps=None, device=None):
    """Eigendecomposition of a symmetric matrix by Jacobi rotations on the GPU;
    sweeps until the off-diagonal Frobenius mass is below tol x ||M||_F (default
    1e-14) or max_sweeps (default 50), then ConvergenceError with the mass
    reached. Eigenvalues descending, ties in their prior column order."""
    arr = as_dense_array(M)
    n, m = arr.shape
    if n != m:
        raise ValueError("symmetric_eig requires a square matrix")
    scale = float(np.max(np.abs(arr))) if arr.size else 0.0
    asym = float(np.max(np.abs(arr - arr.T))) if arr.size else 0.0
    if asym > 1e-10 * max(1.0, scale):
        raise ValueError("matrix is not symmetric to tolerance; symmetrize as (M + M^T)/2 first")
    tol = krylov.JACOBI_TOL if tol is None else tol
    max_sweeps = krylov.JACOBI_MAX_SWEEPS if max_sweeps is None else max_sweeps
    dev = _device(device)
    with torch.cuda.device(dev):
        W = torch.from_numpy(0.5 * (arr + arr.T)).to(device=dev, dtype=torch.float64)
        V = torch.eye(n, dtype=torch.float64, device=dev)
        info, off = ops.jacobi_sweeps(W, V, float(tol), int(max_sweeps))
        info = info.cpu().numpy()
        off = float(off.cpu()[0])
        if not bool(info[0]):
            raise ConvergenceError(f"Jacobi did not converge in {max_sweeps} sweeps (off-diagonal mass {off:.3e})",
                                   residual=off)
        vals = torch.diagonal(W).cpu().numpy().copy()
        vecs = V.cpu().numpy()
    order = np.argsort(-vals, kind="stable")
    return EigResult(vals[order], DenseMatrix(np.ascontiguousarray(vecs[:, order])))


ORACLE_DIM_LIMIT = 2000  # factor.py:36


@dataclass(frozen=True)
class SvdResult:
    """factor.py:59-76 -- thin SVD factors: U (n x r), singular values
    descending, V (d x r)."""

    U: DenseMatrix
    singular_values: np.ndarray
    V: DenseMatrix

    def __post_init__(self):
        sv = np.array(self.singular_values, dtype=np.float64, copy=True)
        if sv.ndim != 1 or np.any(sv < 0) or np.any(np.diff(sv) > 0):
            raise ValueError("singular values must be nonnegative and descending")
        sv.setflags(write=False)
        object.__setattr__(self, "singular_values", sv)

    @property
    def rank(self):
        return int(self.singular_values.shape[0])


def dense_svd_reference(A, dim_limit=ORACLE_DIM_LIMIT, device=None):
    """factor.py:169-214 -- the desk-scale oracle SVD through the smaller Gram
    matrix and symmetric_eig, refused above the guard; directions below 1e-12 of
    the largest singular value are dropped. Products and the eigensolve run on
    the GPU (FP64)."""
    from .matrix import as_operator, matmul

    op = as_operator(A)
    n, d = op.shape
    if min(n, d) > dim_limit:
        raise ValueError(f"reference SVD guard: min(n, d) = {min(n, d)} exceeds {dim_limit}; "
                         "supply a cached oracle or reduce the problem size")
    dense = op.densify().data
    via_transpose = d > n
    left = dense if via_transpose else np.ascontiguousarray(dense.T)
    gram = matmul(left, np.ascontiguousarray(left.T)).data
    eig = symmetric_eig(0.5 * (gram + gram.T), device=device)
    small = eig.eigenvectors.data
    sigma = np.sqrt(np.clip(eig.eigenvalues, 0.0, None))
    keep = sigma >= 1e-12 * sigma[0] if (sigma.size and sigma[0] > 0.0) else np.zeros(sigma.shape, dtype=bool)
    sigma = sigma[keep]
    kept = np.ascontiguousarray(small[:, keep])
    if sigma.size:
        if via_transpose:
            u = kept
            v = matmul(np.ascontiguousarray(dense.T), u).data / sigma[None, :]
        else:
            v = kept
            u = matmul(dense, v).data / sigma[None, :]
    else:
        u, v = np.zeros((n, 0)), np.zeros((d, 0))
    return SvdResult(DenseMatrix(u), sigma, DenseMatrix(v))


def spectral_norm_est(op, tol=1e-9, max_iters=10000, rng=None, device=None):
    """factor.py:217-253 -- power-iteration estimate of the largest singular
    value (a lower bound: the largest Rayleigh estimate seen from a Gaussian
    start, stopped when successive estimates agree to ``tol`` relative). ``op``:
    a matrix or the operator handle; the products run on the GPU."""
    from .matrix import SeededRng, as_operator
    from .metrics import _Plain, spectral_norm_batched

    if tol <= 0:
        raise ValueError("tol must be positive")
    if rng is None:
        rng = SeededRng(0)
    mop = as_operator(op)
    start = rng.normal_fill(mop.shape[1]).reshape(-1, 1)
    dop = mop.device_operator()
    with torch.cuda.device(dop.device):
        best, _ = spectral_norm_batched(_Plain(dop), tol=tol, max_iters=max_iters, starts=start)
    return float(best[0])


def spectral_norm_max_restarts(op, tol=1e-9, max_iters=10000, seeds=(101, 202, 303)):
    """factor.py:256-261 -- max of spectral_norm_est over independent seeded
    starts (batched as columns of one block: one pass over A per iteration)."""
    from .matrix import as_operator
    from .metrics import _Plain, spectral_norm_batched

    dop = as_operator(op).device_operator()
    with torch.cuda.device(dop.device):
        best, _ = spectral_norm_batched(_Plain(dop), seeds=tuple(seeds), tol=tol, max_iters=max_iters)
    return float(best.max())
