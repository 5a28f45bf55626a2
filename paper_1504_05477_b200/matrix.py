"""Host-side matrix containers and the seeded Gaussian source — the
reference's public types on this path (matrix.py:38-309), same validation
and error behaviour, plus device-side upload helpers.

``SeededRng`` draws through the C ABI's host stream (rsvd_gauss_fill), bit
for bit the reference's SplitMix64 + Box-Muller stream.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_MASK64 = (1 << 64) - 1


class SeededRng:
    """matrix.py:38-70 — deterministic Gaussian stream; equal seeds give
    bitwise-equal streams; a fill of m normals consumes 2*ceil(m/2) uniforms."""

    def __init__(self, seed):
        seed = int(seed)
        if not 0 <= seed <= _MASK64:
            raise ValueError("seed must fit in an unsigned 64-bit integer")
        self.seed = seed
        self._state = seed

    def normal_fill(self, count):
        if count < 0:
            raise ValueError("count must be nonnegative")
        from .device import gauss_fill_host

        out, self._state = gauss_fill_host(int(count), self._state)
        return out

    def normal(self):
        return float(self.normal_fill(1)[0])


@dataclass(frozen=True)
class DenseMatrix:
    """matrix.py:73-98 — row-major float64, finite, read-only."""

    data: np.ndarray

    def __post_init__(self):
        arr = np.array(self.data, dtype=np.float64, order="C", copy=True)
        if arr.ndim != 2:
            raise ValueError("dense matrix data must be 2-D")
        if not np.all(np.isfinite(arr)):
            raise ValueError("dense matrix entries must be finite")
        arr.setflags(write=False)
        object.__setattr__(self, "data", arr)

    @property
    def rows(self):
        return self.data.shape[0]

    @property
    def cols(self):
        return self.data.shape[1]

    @property
    def shape(self):
        return self.data.shape


@dataclass(frozen=True)
class SparseMatrixCSR:
    """matrix.py:101-185 — CSR with non-decreasing row pointer, strictly
    increasing columns within a row, finite nonzero values."""

    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        rows, cols = int(self.rows), int(self.cols)
        if rows < 1 or cols < 1:
            raise ValueError("sparse matrix dimensions must be positive")
        rp = np.array(self.row_ptr, dtype=np.int64, order="C", copy=True)
        ci = np.array(self.col_idx, dtype=np.int64, order="C", copy=True)
        vv = np.array(self.values, dtype=np.float64, order="C", copy=True)
        if rp.ndim != 1 or rp.shape[0] != rows + 1:
            raise ValueError("row_ptr must have length rows + 1")
        nnz = ci.shape[0]
        if vv.shape[0] != nnz:
            raise ValueError("col_idx and values must have equal length")
        if rp[0] != 0 or rp[-1] != nnz or np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr must be non-decreasing from 0 to nnz")
        if nnz:
            if ci.min() < 0 or ci.max() >= cols:
                raise ValueError("column index out of bounds")
            if not np.all(np.isfinite(vv)) or np.any(vv == 0.0):
                raise ValueError("values must be finite and nonzero")
            # strictly increasing within each row: a non-increase is allowed
            # only where a new row starts
            row_starts = np.zeros(nnz, dtype=bool)
            row_starts[rp[1:-1][(rp[1:-1] > 0) & (rp[1:-1] < nnz)]] = True
            if nnz > 1 and not np.all((np.diff(ci) > 0) | row_starts[1:]):
                raise ValueError("column indices must strictly increase within a row")
        for a in (rp, ci, vv):
            a.setflags(write=False)
        object.__setattr__(self, "rows", rows)
        object.__setattr__(self, "cols", cols)
        object.__setattr__(self, "row_ptr", rp)
        object.__setattr__(self, "col_idx", ci)
        object.__setattr__(self, "values", vv)

    @property
    def nnz(self):
        return int(self.values.shape[0])

    @property
    def shape(self):
        return (self.rows, self.cols)

    @classmethod
    def from_coo(cls, rows, cols, row_indices, col_indices, values):
        """matrix.py:157-178 — duplicates summed, explicit zeros dropped."""
        ri = np.asarray(row_indices, dtype=np.int64)
        ci = np.asarray(col_indices, dtype=np.int64)
        vv = np.asarray(values, dtype=np.float64)
        if ri.size:
            keys = ri * int(cols) + ci
            uniq, inverse = np.unique(keys, return_inverse=True)
            summed = np.zeros(uniq.shape[0], dtype=np.float64)
            np.add.at(summed, inverse, vv)
            keep = summed != 0.0
            uniq, vv = uniq[keep], summed[keep]
            ri, ci = uniq // int(cols), uniq % int(cols)
        counts = np.bincount(ri, minlength=int(rows)) if ri.size else np.zeros(int(rows), dtype=np.int64)
        row_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        return cls(rows, cols, row_ptr, ci, vv)

    def toarray(self):
        out = np.zeros((self.rows, self.cols), dtype=np.float64)
        r = np.repeat(np.arange(self.rows), np.diff(self.row_ptr))
        out[r, self.col_idx] = self.values
        return out


def as_dense_array(m):
    """matrix.py:188-192."""
    if isinstance(m, DenseMatrix):
        return m.data
    return DenseMatrix(np.asarray(m)).data


def gaussian(rows, cols, rng):
    """matrix.py:266-276 — rows x cols standard normals, filled row-major."""
    rows, cols = int(rows), int(cols)
    if rows < 1 or cols < 1:
        raise ValueError("gaussian dimensions must be at least 1")
    return DenseMatrix(rng.normal_fill(rows * cols).reshape(rows, cols))


class MatrixOperator:
    """matrix.py:195-257 -- uniform apply / apply-transpose access over dense or
    CSR storage, numpy in / numpy out like the reference's. The matrix is
    uploaded once (FP64, on first use) and stays resident on the device; the
    products run in librsvd_b200.so (FP64 tensor-core GEMMs / CSR kernels)."""

    def __init__(self, matrix):
        if isinstance(matrix, MatrixOperator):
            matrix = matrix.matrix
        if isinstance(matrix, (DenseMatrix, SparseMatrixCSR)):
            self.matrix = matrix
        else:
            self.matrix = DenseMatrix(np.asarray(matrix))
        self._dev = None

    @property
    def shape(self):
        return self.matrix.shape

    @property
    def is_sparse(self):
        return isinstance(self.matrix, SparseMatrixCSR)

    @property
    def nnz(self):
        if self.is_sparse:
            return self.matrix.nnz
        return int(np.count_nonzero(self.matrix.data))

    def device_operator(self):
        """The device-resident operator behind this one (operators.py)."""
        if self._dev is None:
            from .rsvd import make_operator

            self._dev = make_operator(self.matrix, precision="fp64")
        return self._dev

    def _product(self, block, inner, rows_out, transpose):
        import torch

        b = np.ascontiguousarray(np.asarray(block, dtype=np.float64))
        if b.ndim == 1:
            b = b.reshape(-1, 1)
        if b.shape[0] != inner:
            raise ValueError("inner dimensions do not match")
        op = self.device_operator()
        with torch.cuda.device(op.device):
            x = torch.from_numpy(b).to(op.device)
            out = torch.empty((rows_out, b.shape[1]), dtype=torch.float64, device=op.device)
            if b.shape[1]:
                (op.apply_t if transpose else op.apply)(x, out)
            return out.cpu().numpy()

    def apply(self, block):
        """A @ block."""
        return self._product(block, self.shape[1], self.shape[0], False)

    def apply_transpose(self, block):
        """A.T @ block."""
        return self._product(block, self.shape[0], self.shape[1], True)

    def densify(self):
        if self.is_sparse:
            return DenseMatrix(self.matrix.toarray())
        return self.matrix

    def frobenius_sq(self):
        from .metrics import frobenius_sq

        return frobenius_sq(self.device_operator())


def as_operator(A):
    """matrix.py:260-263."""
    if isinstance(A, MatrixOperator):
        return A
    return MatrixOperator(A)


def matmul(A, B):
    """matrix.py:279-287 -- dense product A @ B (FP64 tensor-core GEMM;
    fixed summation order: bitwise reproducible)."""
    from . import backend

    a = as_dense_array(A)
    b = as_dense_array(B)
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"matmul dimension mismatch: {a.shape} x {b.shape}")
    return DenseMatrix(backend.mm(a, b))


def spmm(A, B, transpose_A=False):
    """matrix.py:290-304 -- sparse-dense product A @ B, or A.T @ B."""
    from . import backend

    if not isinstance(A, SparseMatrixCSR):
        raise TypeError("spmm expects a SparseMatrixCSR left operand")
    b = as_dense_array(B)
    inner = A.rows if transpose_A else A.cols
    if b.shape[0] != inner:
        raise ValueError(f"spmm dimension mismatch: {A.shape}{'^T' if transpose_A else ''} x {b.shape}")
    if transpose_A:
        out = backend.spmm_t(A.rows, A.cols, A.row_ptr, A.col_idx, A.values, b)
    else:
        out = backend.spmm_nt(A.rows, A.row_ptr, A.col_idx, A.values, b)
    return DenseMatrix(out)


def frobenius_norm_sq(A):
    """matrix.py:307-309 -- sum of squared entries."""
    return as_operator(A).frobenius_sq()
