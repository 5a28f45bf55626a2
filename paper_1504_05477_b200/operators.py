"""Device-resident operators: the B200 counterpart of MatrixOperator
(matrix.py:195-257). ``apply`` is A X, ``apply_t`` is A^T Y (a partial sum
over the local rows when A is row-sharded; the caller allreduces).

Dense A is read in place for both products (the reference caches a
contiguous A^T copy, matrix.py:245-247). Implicit mean-centering (PCA) is a
rank-1 correction folded into the GEMM epilogues:
    (A - 1 mu^T) X   = A X   - 1 (mu^T X)
    (A - 1 mu^T)^T Y = A^T Y - mu (1^T Y)
with mu the column means of the full (all-rank) matrix, kept in FP64.
"""

from __future__ import annotations

import torch

from . import device as ops


class DenseDeviceOp:
    def __init__(self, A, n_total=None, row_offset=0, center=False, comm=None):
        if A.dim() != 2 or not A.is_cuda:
            raise ValueError("DenseDeviceOp needs a 2-D CUDA tensor")
        if A.dtype not in (torch.float32, torch.float64):
            raise ValueError(f"unsupported dtype {A.dtype}")
        self.A = A if A.stride(1) == 1 else A.contiguous()
        self.local_rows = A.shape[0]
        self.n_total = A.shape[0] if n_total is None else int(n_total)
        self.row_offset = int(row_offset)
        self.shape = (self.n_total, A.shape[1])
        self.dtype = A.dtype
        self.device = A.device
        self.mu = None
        if center:
            mu = ops.colreduce(self.A, square=False)
            if comm is not None:
                comm.allreduce(mu)
            self.mu = mu / float(self.n_total)
            self._mu_col = self.mu.view(-1, 1)

    def set_column_sums(self, sums):
        """Re-derive mu in place from the (all-rank) column sums of a freshly
        uploaded A (the persistent buffer of a cached graph keeps its mu
        tensor, so a captured factorization sees the new mean)."""
        torch.div(sums, float(self.n_total), out=self.mu)

    @property
    def is_sparse(self):
        return False

    def apply(self, X, out):
        row_sub = None
        if self.mu is not None:
            X64 = X if X.dtype == torch.float64 else ops.convert(X, torch.empty(X.shape, dtype=torch.float64,
                                                                               device=X.device))
            row_sub = torch.empty((1, X.shape[1]), dtype=torch.float64, device=X.device)
            ops.gemm_tn(self._mu_col, X64, row_sub)
        if out.dtype == self.dtype:
            return ops.gemm_nn(self.A, X, out, row_sub=row_sub)
        tmp = torch.empty(out.shape, dtype=self.dtype, device=out.device)
        ops.gemm_nn(self.A, X, tmp, row_sub=row_sub)
        return ops.convert(tmp, out)

    def apply_t(self, Y, out):
        mu = cs = None
        if self.mu is not None:
            # 1^T Y over the LOCAL rows; the caller's allreduce of out sums the
            # partial (A_g^T Y_g - mu 1^T Y_g) terms into the full correction.
            cs = ops.colreduce(Y, square=False)
            mu = self.mu
        return ops.gemm_tn(self.A, Y, out, mu=mu, colsum_b=cs)


class CsrDeviceOp:
    """CSR A on the device; A^T products run as a gather over the CSR of A^T
    built once (spmm_t, _kernels.pyx:95-113, without atomics). Both products
    go through row-split plans (ops.SpmmPlan) so that the long rows of A^T
    (Zipf-heavy columns of A) are spread over many warps."""

    def __init__(self, indptr, col, val, ncols, n_total=None, row_offset=0):
        self.indptr, self.col, self.val = indptr, col, val
        nrows = indptr.numel() - 1
        self.local_rows = nrows
        self.ncols = int(ncols)
        self.n_total = nrows if n_total is None else int(n_total)
        self.row_offset = int(row_offset)
        self.shape = (self.n_total, self.ncols)
        self.dtype = val.dtype
        self.device = val.device
        self.t_indptr, self.t_col, self.t_val = ops.csr_transpose(indptr, col, val, nrows, self.ncols)
        self.plan = ops.SpmmPlan(indptr)
        self.t_plan = ops.SpmmPlan(self.t_indptr)
        self.mu = None

    @property
    def is_sparse(self):
        return True

    @property
    def nnz(self):
        return self.val.numel()

    def apply(self, X, out):
        if out.dtype == self.dtype:
            return ops.spmm_csr_plan(self.plan, self.col, self.val, X, out)
        tmp = torch.empty(out.shape, dtype=self.dtype, device=out.device)
        ops.spmm_csr_plan(self.plan, self.col, self.val, X, tmp)
        return ops.convert(tmp, out)

    def apply_t(self, Y, out):
        if out.dtype == self.dtype:
            return ops.spmm_csr_plan(self.t_plan, self.t_col, self.t_val, Y, out)
        tmp = torch.empty(out.shape, dtype=self.dtype, device=out.device)
        ops.spmm_csr_plan(self.t_plan, self.t_col, self.t_val, Y, tmp)
        return ops.convert(tmp, out)
