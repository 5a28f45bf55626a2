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

import os

import torch

from . import device as ops

# Exact mode: Rayleigh-Ritz W = A^T Q with reduced digit levels
# (RSVD_OZ_REDUCED_RR=0: full accuracy, for A/B measurement).
OZ_REDUCED_RR = os.environ.get("RSVD_OZ_REDUCED_RR", "1") != "0"
# FP32 CSR products on the nonzero-balanced plan (RSVD_SPMM_ROWPLAN=1: the
# warp-per-row plan, for A/B measurement).
NNZ_PLAN = os.environ.get("RSVD_SPMM_ROWPLAN", "0") != "1"
NNZ_PLAN_T = os.environ.get("RSVD_SPMM_NNZ_T", "0") == "1"


class DenseDeviceOp:
    """``exact=True`` (FP32 A only): the Krylov blocks are FP64 and both
    products are FP64-accurate int8 tensor-core GEMMs (Ozaki digit planes of
    A, csrc/gemm_oz.cu) -- the reference's float64 arithmetic on an A that
    stays FP32 in HBM. ``prepare()`` (called at the start of every
    factorization, inside its CUDA graph) re-cuts the digit planes from A."""

    def __init__(self, A, n_total=None, row_offset=0, center=False, comm=None, exact=False):
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
        self.oz = None
        # True: the caller cuts the digit planes itself (rsvd._run cuts each row
        # panel as its upload lands), prepare() leaves them alone
        self.external_planes = False
        if exact:
            if A.dtype != torch.float32:
                raise ValueError("exact (Ozaki) products are for FP32 A; FP64 A uses FP64 products already")
            self.oz = ops.OzPlanes(self.A)
            self.dtype = torch.float64  # work precision of the Krylov blocks
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

    def prepare(self):
        """Per-factorization setup on the stream (exact mode: digit planes)."""
        if self.oz is not None and not self.external_planes:
            self.oz.refresh(self.A)

    def apply(self, X, out):
        if self.oz is not None:
            ops.oz_gemm(self.oz, X, out, trans=0)
            if self.mu is not None:
                # (A - 1 mu^T) X = A X - 1 (mu^T X), all FP64
                row_sub = torch.empty((1, X.shape[1]), dtype=torch.float64, device=X.device)
                ops.gemm_tn(self._mu_col, X, row_sub)
                ops.gemm_nn(self._ones_col(), row_sub, out, alpha=-1.0, beta=1.0)
            return out
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

    def _ones_col(self):
        if getattr(self, "_ones", None) is None:
            self._ones = torch.ones((self.local_rows, 1), dtype=torch.float64, device=self.device)
        return self._ones

    def apply_t(self, Y, out, rayleigh_ritz=False):
        """``rayleigh_ritz`` (exact mode): W = A^T Q of post_process at ~3e-11
        relative accuracy (reduced digit levels); W's error enters the Ritz
        values linearly, unlike the Krylov chain's, which the reference's
        power-block basis amplifies ~1e9-fold."""
        if self.oz is not None:
            ops.oz_gemm(self.oz, Y, out, trans=1, reduced=rayleigh_ritz and OZ_REDUCED_RR)
            if self.mu is not None:
                # (A - 1 mu^T)^T Y = A^T Y - mu (1^T Y) over the local rows
                cs = ops.colreduce(Y, square=False).view(1, -1)
                ops.gemm_nn(self._mu_col, cs, out, alpha=-1.0, beta=1.0)
            return out
        mu = cs = None
        if self.mu is not None:
            # 1^T Y over the LOCAL rows; the caller's allreduce of out sums the
            # partial (A_g^T Y_g - mu 1^T Y_g) terms into the full correction.
            cs = ops.colreduce(Y, square=False)
            mu = self.mu
        # Y's split planes, when the product that wrote Y left them behind
        return ops.gemm_tn(self.A, Y, out, mu=mu, colsum_b=cs, b_planes=ops.SplitPlanes.peek(Y.device))


class CsrDeviceOp:
    """CSR A on the device; A^T products run as a gather over the CSR of A^T
    built once (spmm_t, _kernels.pyx:95-113, without atomics). Both products
    go through row-split plans (ops.SpmmPlan) so that the long rows of A^T
    (Zipf-heavy columns of A) are spread over many warps.

    Hybrid hot/cold split (FP32): a CSR product is gather-bound -- every
    nonzero reads one b-wide row of the dense block from L2, ~400 bytes at
    b = 100 against 8 bytes of A. Columns holding at least `hot_density` x
    rows nonzeros (the Zipf head of C3: ~0.1% of the columns, ~40% of the
    nonzeros) are stored once as a dense row-major panel A_hot (rows x H,
    zeros included) and multiplied on the tensor cores (3xTF32 GEMM:
    A_hot X[hot] and A_hot^T Y), the remaining nonzeros stay CSR:
        A X   = A_hot X[hot] + A_cold X
        A^T Y = scatter(hot, A_hot^T Y) + A_cold^T Y   (hot rows of A_cold^T empty)
    A dense column costs 2 rows b flops on the tensor pipe; its nonzeros cost
    nnz_j b 4 bytes of L2 gather, so a column pays off above ~3% density."""

    HOT_DENSITY = float(os.environ.get("RSVD_SPMM_HOT_DENSITY", "0.03"))
    HOT_MAX = 2048
    # Slab tier (A X only): the next SLAB_COLS most frequent columns keep their
    # rows of X in shared memory (csrc/sparse.cu k_spmm_slab); 2048 columns x
    # a 25-column chunk of the block fill one SM's 200 KB. A column is worth a
    # slab row when every row group meets it several times: at least
    # SLAB_MIN_COUNT nonzeros. OFF by default (RSVD_SPMM_SLAB_COLS=2048 turns it
    # on): measured at C3 the tier takes 21 % of the nonzeros off the L2 gather
    # (0.62 -> 0.47 ms) but its own pass costs 0.37 ms -- rows hold ~21 slab
    # nonzeros each, so the per-row pointer / index / C read-modify-write
    # latency, not shared-memory bandwidth, sets its pace (SpMM).
    SLAB_COLS = int(os.environ.get("RSVD_SPMM_SLAB_COLS", "0"))
    SLAB_MIN_COUNT = 64

    def __init__(self, indptr, col, val, ncols, n_total=None, row_offset=0, hot_density=None):
        nrows = indptr.numel() - 1
        self.local_rows = nrows
        self.ncols = int(ncols)
        self.n_total = nrows if n_total is None else int(n_total)
        self.row_offset = int(row_offset)
        self.shape = (self.n_total, self.ncols)
        self.dtype = val.dtype
        self.device = val.device
        self.mu = None
        self._nnz = val.numel()
        dens = self.HOT_DENSITY if hot_density is None else float(hot_density)
        self.hot = None
        if val.dtype == torch.float32 and dens > 0 and nrows >= 128 and val.numel() > 0:
            self.hot = self._split_hot(indptr, col, val, nrows, dens)
        if self.hot is not None:
            indptr, col, val = self.hot["cold"]
        # A^T Y gathers over every non-hot nonzero; A X takes the slab columns out as well
        self.t_indptr, self.t_col, self.t_val = ops.csr_transpose(indptr, col, val, nrows, self.ncols)
        self.t_plan = ops.SpmmPlan(self.t_indptr)
        self.slab = None
        if val.dtype == torch.float32 and self.SLAB_COLS > 0 and nrows >= 128 and val.numel() > 0:
            self.slab = self._split_slab(indptr, col, val, nrows)
        if self.slab is not None:
            indptr, col, val = self.slab.pop("cold")
        self.indptr, self.col, self.val = indptr, col, val
        self.plan = ops.SpmmPlan(indptr)
        # nonzero-balanced plans of the FP32 fast path, built on first use
        self._nnz_plan = self._nnz_plan_t = None

    def prepare(self):
        """Per-factorization setup (nothing for CSR)."""

    def _split_hot(self, indptr, col, val, nrows, dens):
        """Operator setup (torch plumbing, once): pick the hot columns, build
        the dense panel and the cold CSR (nonzero order kept)."""
        counts = torch.bincount(col.to(torch.int64), minlength=self.ncols)
        thr = max(1, int(dens * nrows))
        hot = torch.nonzero(counts >= thr).flatten()
        if hot.numel() == 0:
            return None
        if hot.numel() > self.HOT_MAX:
            hot = hot[torch.argsort(counts[hot], descending=True)[: self.HOT_MAX]].sort().values
        H = hot.numel()
        Hp = (H + 3) // 4 * 4  # 16-byte rows for the tensor-core operand
        pos = torch.full((self.ncols,), -1, dtype=torch.int64, device=col.device)
        pos[hot] = torch.arange(H, device=col.device)
        ip = indptr.to(torch.int64)
        rows = torch.repeat_interleave(torch.arange(nrows, device=col.device), ip[1:] - ip[:-1])
        pcol = pos[col.to(torch.int64)]
        is_hot = pcol >= 0
        panel = torch.zeros((nrows, Hp), dtype=val.dtype, device=val.device)
        panel[rows[is_hot], pcol[is_hot]] = val[is_hot]
        cold = ~is_hot
        cold_counts = torch.bincount(rows[cold], minlength=nrows)
        cptr = torch.zeros(nrows + 1, dtype=indptr.dtype, device=indptr.device)
        cptr[1:] = torch.cumsum(cold_counts, 0).to(indptr.dtype)
        return {"idx": hot.contiguous(), "H": H, "Hp": Hp, "panel": panel,
                "cold": (cptr, col[cold].contiguous(), val[cold].contiguous()),
                "hot_nnz": int(is_hot.sum())}

    def _split_slab(self, indptr, col, val, nrows):
        """Operator setup (torch plumbing, once): the most frequent remaining
        columns as a CSR over slab row indices, and the CSR without them."""
        counts = torch.bincount(col.to(torch.int64), minlength=self.ncols)
        m = min(self.SLAB_COLS, self.ncols)
        top = torch.topk(counts, m)
        keep = top.values >= self.SLAB_MIN_COUNT
        cols = top.indices[keep].sort().values
        if cols.numel() == 0:
            return None
        pos = torch.full((self.ncols,), -1, dtype=torch.int64, device=col.device)
        pos[cols] = torch.arange(cols.numel(), device=col.device)
        ip = indptr.to(torch.int64)
        rows = torch.repeat_interleave(torch.arange(nrows, device=col.device), ip[1:] - ip[:-1])
        pcol = pos[col.to(torch.int64)]
        in_slab = pcol >= 0

        def ptr_of(sel):
            c = torch.bincount(rows[sel], minlength=nrows)
            p = torch.zeros(nrows + 1, dtype=torch.int32, device=col.device)
            p[1:] = torch.cumsum(c, 0).to(torch.int32)
            return p

        cold = ~in_slab
        cptr = ptr_of(cold).to(indptr.dtype)
        return {"ptr": ptr_of(in_slab), "idx": pcol[in_slab].to(torch.int32).contiguous(),
                "val": val[in_slab].contiguous(), "cols": cols.contiguous(), "nnz": int(in_slab.sum()),
                "cold": (cptr, col[cold].contiguous(), val[cold].contiguous())}

    @property
    def is_sparse(self):
        return True

    @property
    def nnz(self):
        return self._nnz

    def _x_hot(self, X):
        h = self.hot
        xh = torch.zeros((h["Hp"], X.shape[1]), dtype=X.dtype, device=X.device)
        ops.gather_rows(h["idx"], X, xh[: h["H"]])
        return xh

    def _gather(self, trans, B, C, beta=0.0):
        """The CSR part of a product: the nonzero-balanced kernel when the
        block qualifies (FP32, int32 indices, width <= 128 and a multiple of
        4, 16-byte rows), else warp-per-row chunks (RSVD_SPMM_ROWPLAN=1
        forces those, for A/B measurement)."""
        col, val = (self.t_col, self.t_val) if trans else (self.col, self.val)
        # A^T Y stays on the row plan: the rows of A^T (columns of A) are mostly a
        # handful of nonzeros, where a run of 256 nonzeros is a string of row
        # flushes (measured at C3: 0.54 ms against 0.44 ms; A X 0.55 against 0.61)
        if NNZ_PLAN and (not trans or NNZ_PLAN_T) and ops.SpmmNnzPlan.eligible(col, val, B, C):
            if trans:
                if self._nnz_plan_t is None:
                    self._nnz_plan_t = ops.SpmmNnzPlan(self.t_indptr)
                plan = self._nnz_plan_t
            else:
                if self._nnz_plan is None:
                    self._nnz_plan = ops.SpmmNnzPlan(self.indptr)
                plan = self._nnz_plan
            return ops.spmm_nnz_plan(plan, col, val, B, C, beta=beta)
        return ops.spmm_csr_plan(self.t_plan if trans else self.plan, col, val, B, C, beta=beta)

    def _apply32(self, X, out):
        if self.hot is None:
            self._gather(0, X, out)
        else:
            ops.gemm_nn(self.hot["panel"], self._x_hot(X), out)
            self._gather(0, X, out, beta=1.0)
        if self.slab is not None:
            ops.spmm_slab(self.slab, X, out)
        return out

    def _apply_t32(self, Y, out):
        self._gather(1, Y, out)
        if self.hot is not None:
            h = self.hot
            th = torch.empty((h["Hp"], Y.shape[1]), dtype=out.dtype, device=out.device)
            ops.gemm_tn(h["panel"], Y, th, b_planes=ops.SplitPlanes.peek(Y.device))
            ops.scatter_rows(h["idx"], th[: h["H"]], out)
        return out

    def apply(self, X, out):
        if out.dtype == self.dtype and X.dtype == self.dtype:
            return self._apply32(X, out) if self.dtype == torch.float32 else \
                ops.spmm_csr_plan(self.plan, self.col, self.val, X, out)
        tmp = torch.empty(out.shape, dtype=self.dtype, device=out.device)
        if self.dtype == torch.float32:
            self._apply32(X, tmp)
        else:
            ops.spmm_csr_plan(self.plan, self.col, self.val, X, tmp)
        return ops.convert(tmp, out)

    def apply_t(self, Y, out):
        if out.dtype == self.dtype and Y.dtype == self.dtype:
            return self._apply_t32(Y, out) if self.dtype == torch.float32 else \
                ops.spmm_csr_plan(self.t_plan, self.t_col, self.t_val, Y, out)
        tmp = torch.empty(out.shape, dtype=self.dtype, device=out.device)
        if self.dtype == torch.float32:
            self._apply_t32(Y, tmp)
        else:
            ops.spmm_csr_plan(self.t_plan, self.t_col, self.t_val, Y, tmp)
        return ops.convert(tmp, out)
