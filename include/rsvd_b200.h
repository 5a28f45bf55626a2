/*
 * rsvd_b200 — C ABI of the B200-native randomized block-Krylov partial SVD.
 *
 * Drop-in boundary for the reference package rsvdkit 0.1.0
 * (/root/reference/pkg/src/rsvdkit). The reference binds one kernel module at
 * import (backend.py:39-43) with five entry points; each has a counterpart
 * here, plus the blocked device operations that replace the numpy BLAS-2
 * column loop of _mgs (factor.py:93-98) and the Rayleigh-Ritz post-process
 * (rsvd.py:200-221).
 *
 * Conventions
 *   - All matrices are row-major with an explicit leading dimension in
 *     elements. Device pointers are plain addresses (owned by the caller,
 *     e.g. torch tensors); `stream` is a cudaStream_t (NULL = legacy stream).
 *   - Every device entry point is stream-ordered and asynchronous: it only
 *     enqueues work. Outputs are caller-allocated. Scratch space is an
 *     explicit caller-provided workspace whose size a *_ws_bytes query gives.
 *   - dtype codes: RSVD_F32 / RSVD_F64. Small (p x p, w x w) matrices are
 *     always FP64.
 *   - Status: RSVD_OK, RSVD_ERR_INVALID (host maps to ValueError),
 *     RSVD_ERR_CONVERGENCE (ConvergenceError, errors.py:14-23),
 *     RSVD_ERR_CUDA (RuntimeError). rsvd_last_error() holds the message
 *     (thread-local).
 *   - Results are bitwise deterministic for a fixed device model, shape and
 *     stream: every reduction has a fixed order; no floating-point atomics.
 *   - `pred` (nullable, device int32): when given, the operation's kernels
 *     run only if *pred != 0 and are otherwise no-ops. This lets the host
 *     enqueue data-dependent steps (the second deflation round) without a
 *     host synchronisation, so a whole factorization can be one CUDA graph.
 */
#ifndef RSVD_B200_H
#define RSVD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSVD_OK 0
#define RSVD_ERR_INVALID 1
#define RSVD_ERR_CONVERGENCE 2
#define RSVD_ERR_CUDA 3

#define RSVD_F32 0
#define RSVD_F64 1

/* GEMM algorithm selector (rsvd_gemm_nn / rsvd_gemm_tn `algo`). */
#define RSVD_GEMM_AUTO 0       /* FP32: 3xTF32 / skinny / SIMT by shape; FP64: DMMA */
#define RSVD_GEMM_SIMT 1       /* CUDA-core FFMA/DFMA, FP32 or FP64 */
#define RSVD_GEMM_TC_3XTF32 2  /* tcgen05 kind::tf32, hi/lo split, FP32 only */
#define RSVD_GEMM_DMMA 3       /* mma.sync f64 (DMMA), FP64 only */
#define RSVD_GEMM_SKINNY 4     /* FP32 CUDA-core, outputs <= 64 columns (orthonormalization sizes) */

const char *rsvd_last_error(void);
int rsvd_abi_version(void);
/* Number of SMs of the current device (grid sizing is derived from it). */
int rsvd_sm_count(void);

/* ---- 1. Gaussian stream (HOST) -----------------------------------------
 * Replaces gauss_fill (_kernels.pyx:31-53; numpy twin _kernels_py.py:27-45):
 * SplitMix64 + Box-Muller, bitwise identical to the reference on the same
 * glibc (compiled with the reference's -ffp-contract=off -fno-builtin-sin
 * -fno-builtin-cos). Writes `count` doubles, returns the advanced state. The
 * start block Pi and the QR fill stream are host-supplied (north_star). */
int rsvd_gauss_fill(int64_t count, uint64_t state, double *out, uint64_t *new_state);

/* ---- 2. Dense products ---------------------------------------------------
 * Replace mm (_kernels.pyx:56-71) as used by MatrixOperator.apply /
 * apply_transpose (matrix.py:227-247) and post_process (rsvd.py:212-219).
 * The reference forms A^T as a cached contiguous copy (matrix.py:245-247);
 * here A^T products read A in place (rsvd_gemm_tn).
 *
 * rsvd_gemm_nn:  C[m x n] = alpha * (A[m x k] - 1 row_sub?) . B[k x n] + beta * C
 *   `row_sub` (optional, length n, FP64): subtracted as alpha*row_sub[j] from
 *   every row of the product — the implicit-centering rank-1 correction
 *   (A - 1 mu^T) B = A B - 1 (mu^T B) with row_sub = mu^T B.
 * rsvd_gemm_tn:  C[k x n] = alpha * (A^T . B - mu colsum_b^T) + beta * C,
 *   A is m x k, B is m x n, the reduction runs over the long dimension m in a
 *   fixed split order with FP64 partials (workspace from rsvd_gemm_tn_ws_bytes).
 *   `mu` (length k) and `colsum_b` (length n) are optional (both or neither).
 *   out_dtype may differ from dtype (FP32 inputs, FP64 Gram/projection). */
int rsvd_gemm_nn(int dtype, int64_t m, int64_t n, int64_t k, double alpha, const void *A,
                 int64_t lda, const void *B, int64_t ldb, double beta, void *C, int64_t ldc,
                 const double *row_sub, int algo, const int32_t *pred, void *stream);
/* Split planes of an FP32 block (K x N, row pitch ldb) as the B operand of the
 * tcgen05 3xTF32 products: hi = TF32 truncation, lo = rna_tf32(x - hi), k-blocked
 * K-major. rsvd_gemm_nn_f32_emit is rsvd_gemm_nn (FP32) that also writes the
 * planes of its OUTPUT C from the epilogue (*emitted = 1; 0 when the shape took
 * a non-tensor-core path and only C was written), so that a following
 * rsvd_gemm_tn_f32_planes -- rsvd_gemm_tn with B given by its planes, B's row
 * index being the reduction index -- needs no pass over B. Both replace mm
 * (_kernels.pyx:56-71) inside _mgs's projections (factor.py:93-98).
 * rsvd_gemm_tn_f32_planes_ok: 1 when that product's shape runs on the tensor
 * cores (else use rsvd_gemm_tn). */
int64_t rsvd_split_planes_bytes(int64_t K, int64_t N);
int rsvd_split_planes(int64_t K, int64_t N, const float *B, int64_t ldb, float *planes,
                      int64_t planes_bytes, const int32_t *pred, void *stream);
int rsvd_gemm_nn_f32_emit(int64_t m, int64_t n, int64_t k, double alpha, const float *A, int64_t lda,
                          const float *B, int64_t ldb, double beta, float *C, int64_t ldc,
                          const double *row_sub, float *planes, int64_t planes_bytes,
                          int32_t *emitted, const int32_t *pred, void *stream);
int rsvd_gemm_tn_f32_planes(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha,
                            const float *A, int64_t lda, const float *B_planes,
                            int64_t planes_bytes, double beta, void *C, int64_t ldc,
                            const double *mu, const double *colsum_b, void *ws, int64_t ws_bytes,
                            const int32_t *pred, void *stream);
int rsvd_gemm_tn_f32_planes_ok(int64_t m, int64_t n, int64_t k, const float *A, int64_t lda);
int64_t rsvd_gemm_tn_ws_bytes(int dtype, int64_t m, int64_t n, int64_t k, int algo);
int rsvd_gemm_tn(int dtype, int out_dtype, int64_t m, int64_t n, int64_t k, double alpha,
                 const void *A, int64_t lda, const void *B, int64_t ldb, double beta, void *C,
                 int64_t ldc, const double *mu, const double *colsum_b, void *ws,
                 int64_t ws_bytes, int algo, const int32_t *pred, void *stream);

/* ---- 2b. FP64-accurate products of an FP32 A (int8 tensor cores, Ozaki) ---
 * Replace mm (_kernels.pyx:56-71) as called by MatrixOperator.apply /
 * apply_transpose (matrix.py:227-247) when A is held in FP32 but the Krylov
 * blocks are FP64: the reference's own arithmetic (it upcasts A to float64,
 * matrix.py:80) at FP64-class accuracy (~1e-16 relative) from kind::i8
 * tcgen05 MMAs with exact int32 sums.
 * rsvd_oz_prepare cuts A (n x d FP32, row pitch lda) ONCE into
 *   rsvd_oz_num_planes() signed base-256 digit planes (int8; column-blocked
 *   layout planes[i][c / 16][r][c % 16], rsvd_oz_planes_bytes(n, d) bytes in all)
 *   and per-row exponents row_exp[n]; the caller owns both buffers.
 * rsvd_oz_gemm trans = 0: C (n x p) = alpha A X + beta C  (X d x p FP64)
 *              trans = 1: C (d x p) = alpha A^T Y + beta C (Y n x p FP64)
 *   (+2: reduced accuracy, ~1e-10 relative instead of ~1e-14: digit levels
 *   i + j <= 3, 10 instead of 20 digit-pair GEMMs; the Rayleigh-Ritz W = A^T Q)
 *   C is FP64; workspace from rsvd_oz_gemm_ws_bytes(trans & 1, n, d, p). */
int64_t rsvd_oz_planes_bytes(int64_t n, int64_t d);
int rsvd_oz_num_planes(void);
int rsvd_oz_prepare(int64_t n, int64_t d, const float *A, int64_t lda, int8_t *planes, int32_t *row_exp,
                    void *stream);
/* rows [r0, r0 + nr) only (r0 a multiple of 32; A = base of the full matrix):
 * lets the caller cut each row panel as its upload lands (the reference's
 * DenseMatrix copy, matrix.py:73-85, pipelined with the first device pass). */
int rsvd_oz_prepare_rows(int64_t n, int64_t d, int64_t r0, int64_t nr, const float *A, int64_t lda,
                         int8_t *planes, int32_t *row_exp, void *stream);
int64_t rsvd_oz_gemm_ws_bytes(int trans, int64_t n, int64_t d, int64_t p);
int rsvd_oz_gemm(int trans, int64_t n, int64_t d, int64_t p, double alpha, const int8_t *planes,
                 const int32_t *row_exp, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                 void *ws, int64_t ws_bytes, const int32_t *pred, void *stream);

/* The same digit-plane products for an FP64 basis Q (n x w): _mgs's
 * projections v <- v - Q_p (Q_p^T v) (factor.py:93-98) against the
 * already-final prefix Q_p = Q[:, :jp]. rsvd_oz_basis_slice cuts columns
 * [c0, c0 + ncols) of Q into rsvd_oz_basis_planes() digit planes with
 * per-column exponents col_exp[c0 .. c0 + ncols) (planes of
 * rsvd_oz_basis_bytes(n, w) bytes; workspace rsvd_oz_basis_ws_bytes(ncols)),
 * one block at a time as blocks become final.
 * rsvd_oz_gemm_planes is rsvd_oz_gemm on any digit planes (nplanes of them,
 * allocated rows_alloc x cols_alloc, multiples of 128; exponents per row of
 * the planes, or per column when col_scaled = 1) using their leading n x d
 * corner: trans = 1 gives Q_p^T V (d = jp), trans = 0 gives Q_p C. */
int rsvd_oz_basis_planes(void);
int64_t rsvd_oz_basis_bytes(int64_t n, int64_t w);
int64_t rsvd_oz_basis_ws_bytes(int64_t ncols);
int rsvd_oz_basis_slice(int64_t n, int64_t w, const double *Q, int64_t ldq, int64_t c0, int64_t ncols,
                        int8_t *planes, int32_t *col_exp, void *ws, int64_t ws_bytes, void *stream);
int rsvd_oz_gemm_planes(int trans, int64_t n, int64_t d, int64_t p, double alpha, const int8_t *planes, int nplanes,
                        int64_t rows_alloc, int64_t cols_alloc, const int32_t *exps, int col_scaled, const double *B,
                        int64_t ldb, double beta, double *C, int64_t ldc, void *ws, int64_t ws_bytes,
                        const int32_t *pred, void *stream);

/* ---- 3. Sparse products --------------------------------------------------
 * Replace spmm_nt (_kernels.pyx:74-92) and spmm_t (_kernels.pyx:95-113).
 * C[nrows x nb] = alpha * A . B + beta * C for CSR A (nrows x ncols).
 * Index arrays are int32 (idx64 = 0) or int64 (idx64 = 1). spmm_t is this
 * same entry point applied to the CSR of A^T, built once per operator
 * (deterministic gather, no atomics) with rsvd_csr_transpose. */
int rsvd_spmm_csr(int dtype, int idx64, int64_t nrows, int64_t ncols, int64_t nb,
                  const void *indptr, const void *col, const void *val, const void *B,
                  int64_t ldb, double alpha, double beta, void *C, int64_t ldc, void *stream);
/* Load-balanced variant with a row-split plan built once per operator (host
 * plumbing, paper_1504_05477_b200/device.py:spmm_plan): chunk c covers the
 * nonzeros [chunk_lo[c], chunk_hi[c]) of row chunk_row[c]; chunk_slot[c] = -1
 * writes C directly, otherwise the partial sum goes to workspace slot
 * chunk_slot[c] (ws: slots x min(nb, 256) elements; wider blocks run in
 * column panels of 256). Split row s (split_row[s]) sums
 * slots [split_beg[s], split_beg[s+1]) in order, then applies alpha / beta:
 * deterministic, no atomics. Rows with no chunk are not touched. */
int rsvd_spmm_csr_plan(int dtype, int idx64, int64_t nrows, int64_t nb, const void *col, const void *val,
                       const void *B, int64_t ldb, double alpha, double beta, void *C, int64_t ldc,
                       int64_t nchunks, const int64_t *chunk_lo, const int64_t *chunk_hi,
                       const int32_t *chunk_row, const int32_t *chunk_slot, int64_t nsplit,
                       const int32_t *split_row, const int64_t *split_beg, void *ws, int64_t ws_bytes,
                       void *stream);
/* Nonzero-balanced FP32 product C = alpha A B + beta C (int32 indices, width
 * nb <= 128, a multiple of 4; spmm_nt / spmm_t on a CSR, _kernels.pyx:74-113):
 * work unit c = nonzeros [c chunk, (c + 1) chunk) with rowid[e] the row of
 * nonzero e. A row that lies inside one unit is written straight to C; the
 * first / last row of a unit that continues in a neighbouring unit goes to
 * workspace slot head_slot[c] / tail_slot[c] (-1: none), the slots of one row
 * being consecutive: split row s (split_row[s]) sums slots [split_beg[s],
 * split_beg[s + 1]) in order. empty_rows: rows without a nonzero (C = beta C).
 * ws: slots x nb floats. Deterministic, no atomics. */
int rsvd_spmm_nnz_plan(int64_t nnz, int chunk, int64_t nb, const int32_t *col, const float *val,
                       const int32_t *rowid, const float *B, int64_t ldb, double alpha, double beta,
                       float *C, int64_t ldc, const int32_t *head_slot, const int32_t *tail_slot,
                       int64_t nsplit, const int32_t *split_row, const int64_t *split_beg,
                       int64_t nempty, const int32_t *empty_rows, void *ws, int64_t ws_bytes,
                       void *stream);
/* Slab tier of the hybrid CSR product (FP32): C += A_slab X, where A_slab holds
 * the nonzeros of `nslab` chosen columns (slab_cols[s] = the column of slab
 * row s) as a CSR over slab row indices (slab_ptr[nrows + 1], slab_idx,
 * slab_val). The X rows of those columns are staged in shared memory, one
 * column chunk of the block at a time (spmm_nt, _kernels.pyx:74-92, for the
 * columns frequent enough that every SM reuses them). Deterministic. */
int rsvd_spmm_slab(int64_t nrows, int64_t nb, const int32_t *slab_ptr, const int32_t *slab_idx,
                   const float *slab_val, const int64_t *slab_cols, int64_t nslab, const float *X,
                   int64_t ldx, float *C, int64_t ldc, void *stream);
/* CSR (nrows x ncols, sorted columns) -> CSR of the transpose, stable in row
 * order. perm_by_col[e] must be a stable column-sorted permutation of the
 * nonzeros (supplied by the caller's sort); t_indptr has ncols+1 entries. */
int rsvd_csr_transpose(int dtype, int idx64, int64_t nrows, int64_t ncols, int64_t nnz,
                       const void *indptr, const void *col, const void *val,
                       const int64_t *perm_by_col, void *t_indptr, void *t_col, void *t_val,
                       void *stream);

/* ---- 4. Block orthonormalization (replaces _mgs, factor.py:79-118) -------
 * Cholesky of the FP64 Gram G (p x p) of a block, in column order, with
 * deficiency deflation: column j is declared deficient when its residual
 * square norm d_j <= tau2 * ref2[j] (ref2 = the column's squared norm
 * before projection; NULL means ref2[j] = G[j][j]), the analogue of
 * factor.py:105 (`nv <= _DEFICIENCY_RTOL * ref`). Writes Tinv = R^{-1}
 * (upper triangular, p x p, zero row+column at deficient slots), mask[j]
 * (1 = deficient), ndef[0] = number of deficient columns and
 * ndef[1] = running[0] before this call; running[0] (nullable, device) is
 * advanced by ndef[0] so successive blocks of one orthonormalization draw
 * successive fill vectors, as one _mgs call does. `active` (nullable): slots
 * with active[j] == 0 are treated as absent (zero row/column of Tinv, not
 * flagged, not counted) — used by the second deflation round, which re-tests
 * only the columns the first (Gram-resolution) round rejected. */
int64_t rsvd_chol_deflate_ws_bytes(int64_t p);
int rsvd_chol_deflate(int64_t p, const double *G, int64_t ldg, const double *ref2, double tau2,
                      double *Tinv, int64_t ldt, int32_t *mask, int32_t *ndef, int32_t *running,
                      const int32_t *active, void *ws, int64_t ws_bytes, const int32_t *pred,
                      void *stream);
/* X[:, j] = 0 where keep[j] == 0. */
int rsvd_mask_cols(int dtype, int64_t n, int64_t p, void *X, int64_t ldx, const int32_t *keep,
                   const int32_t *pred, void *stream);
/* Replacement columns: X[:, j] = fill vector number (ndef[1] + r_j) for every
 * deficient slot j (r_j = deficient slots before j), rows row_offset ..
 * row_offset+n-1 of an n_total-long vector (row-sharded A), generated on the device
 * from the reference's counter-based stream SeededRng(seed) — one vector of n
 * normals per replaced column from a fresh stream per orthonormalization
 * (factor.py:40, 89-90, 107; seed 0x5EED_F111_0C0F_FEE5). No-op when
 * ndef[0] == 0. rsvd_fill_stream writes the first nvec vectors (nvec x n,
 * FP64) for pinning against the host stream. */
int rsvd_insert_fill(int dtype, int64_t n, int64_t p, void *X, int64_t ldx, const int32_t *mask,
                     const int32_t *ndef, uint64_t seed, int64_t row_offset, int64_t n_total,
                     const int32_t *pred, void *stream);
int rsvd_fill_stream(int64_t n, int64_t nvec, uint64_t seed, double *out, void *stream);

/* ---- 5. Symmetric eigensolver (replaces jacobi_sweeps, _kernels.pyx:127-192,
 * and symmetric_eig, factor.py:132-166) -------------------------------------
 * Parallel (round-robin ordered) two-sided Jacobi, one cooperative
 * persistent kernel. Same stop rule as the reference: off(M) <= tol*||M||_F
 * checked after every sweep, rotation skipped when |a_pq| <= tol*||M||_F*1e-3/n,
 * at most max_sweeps sweeps.
 * rsvd_jacobi_sweeps mirrors the kernel contract: M (n x n) is overwritten
 * with its rotated (diagonalised) form, V (pre-initialised by the caller)
 * accumulates the rotations; info = {converged, sweeps}; off_out[0] = final
 * off-diagonal mass. */
int64_t rsvd_jacobi_ws_bytes(int64_t n);
int rsvd_jacobi_sweeps(int64_t n, double *M, int64_t ldm, double *V, int64_t ldv, double tol,
                       int max_sweeps, int32_t *info, double *off_out, void *ws, int64_t ws_bytes,
                       void *stream);
/* Eigenvalues (diag of the diagonalised M) sorted descending, ties keeping
 * index order (factor.py:164-165); writes the top k values and the matching
 * k columns of V (w x k row-major). order_ws: k int32 of scratch. */
int rsvd_eig_select(int64_t w, const double *Mdiag_src, int64_t ldm, const double *V, int64_t ldv,
                    int64_t k, double *evals, double *evecs, int64_t lde, int32_t *order_ws,
                    void *stream);

/* Top-k eigenpairs of a symmetric w x w FP64 matrix for the Rayleigh-Ritz
 * step of post_process (rsvd.py:217-220 consumes only the top k): Householder
 * tridiagonalisation (one cooperative kernel), Sturm multisection for the k
 * largest eigenvalues, inverse iteration with in-cluster
 * re-orthogonalisation, back-transformation (LAPACK dsyevx structure).
 * evals: k values, descending; evecs: w x k row-major (column i pairs with
 * evals[i], sign arbitrary); info[0] = 1 on success, 0 if an eigenvector
 * iteration broke down (host maps to ConvergenceError). M is not modified.
 * evecs = NULL computes the eigenvalues only (the sweep harness's exact
 * oracle spectrum, factor.py:170-215 dense_svd_reference). */
int64_t rsvd_syev_topk_ws_bytes(int64_t w, int64_t k);
int rsvd_syev_topk(int64_t w, const double *M, int64_t ldm, int64_t k, double *evals, double *evecs,
                   int64_t lde, int32_t *info, void *ws, int64_t ws_bytes, void *stream);

/* ---- 6. Element-wise / reductions (all deterministic) -------------------- */
int64_t rsvd_colreduce_ws_bytes(int64_t n, int64_t p);
/* out[j] = sum_i X[i][j]^2 (square=1) or sum_i X[i][j] (square=0), FP64. */
int rsvd_colreduce(int dtype, int square, int64_t n, int64_t p, const void *X, int64_t ldx,
                   double *out, void *ws, int64_t ws_bytes, void *stream);
/* rsvd.py:192-197: flip column j so its largest-magnitude entry (first on
 * ties) is positive. */
int rsvd_canonicalize_signs(int dtype, int64_t n, int64_t k, void *X, int64_t ldx, void *ws,
                            int64_t ws_bytes, void *stream);
/* Row-sharded sign canonicalization, step 1: per column the signed value at
 * the (first) largest-magnitude entry of the local rows and its GLOBAL row
 * index (local index + row_offset; INT64_MAX when n == 0). Step 2, after the
 * ranks exchange these: rsvd_flip_by_sign negates column j where
 * sign_val[j] < 0. */
int rsvd_col_absargmax(int dtype, int64_t n, int64_t k, const void *X, int64_t ldx,
                       int64_t row_offset, double *out_val, int64_t *out_idx, void *ws,
                       int64_t ws_bytes, void *stream);
int rsvd_flip_by_sign(int dtype, int64_t n, int64_t k, void *X, int64_t ldx,
                      const double *sign_val, void *stream);
int rsvd_convert(int src_dtype, int dst_dtype, int64_t rows, int64_t cols, const void *src,
                 int64_t lds, void *dst, int64_t ldd, const int32_t *pred, void *stream);
/* Row gather dst[i, :] = src[idx[i], :] and scatter dst[idx[i], :] = src[i, :],
 * i < nidx, `cols` columns: the hot-column panel of the hybrid CSR product
 * (X_hot = X[hot] before A_hot X_hot; (A^T Y)[hot] = A_hot^T Y after it).
 * Replace the column slicing MatrixOperator leaves to numpy (matrix.py:227-247). */
int rsvd_gather_rows(int dtype, int64_t nidx, int64_t cols, const int64_t *idx, const void *src,
                     int64_t lds, void *dst, int64_t ldd, void *stream);
int rsvd_scatter_rows(int dtype, int64_t nidx, int64_t cols, const int64_t *idx, const void *src,
                      int64_t lds, void *dst, int64_t ldd, void *stream);
/* out[i] = sqrt(max(in[i], 0)) (rsvd.py:220). */
int rsvd_sqrt_clip(int64_t k, const double *in, double *out, void *stream);
/* max |G - I| of a k x k FP64 matrix -> out[0] (rsvd.py:182-185). */
int rsvd_ortho_error(int64_t k, const double *G, int64_t ldg, double *out, void *stream);

/* ---- Device-predicated sections as CUDA-graph IF nodes -------------------
 * While `stream` is being captured: adds a conditional node whose condition
 * is (*flag != 0) at graph execution, and starts capturing `body_stream` into
 * the node's body; the caller issues the section on `body_stream`, then calls
 * rsvd_cond_end. Not capturing: *opened = 0 and nothing happens (the caller
 * issues the section on `stream`). The sections are the orthonormalization's
 * device-decided branches (factor.py:105-116). */
int rsvd_cond_begin(void *stream, const int32_t *flag, void *body_stream, int32_t *opened);
int rsvd_cond_end(void *body_stream);

/* ---- 8. Per-device handle and communicator injection -----
 * An opaque handle bound to one CUDA device (thread-compatible, not
 * thread-safe) that carries the row-sharded run's communicator. The product
 * needs one collective: the in-place sum-allreduce of every reduction over
 * rows (A^T Y partials, Grams, projection coefficients, W = A^T Q).
 * Inject an existing ncclComm_t (rsvd_handle_set_comm; the caller keeps
 * ownership) or build one from a NCCL unique id distributed by the caller
 * (rsvd_nccl_unique_id on one rank, rsvd_handle_init_comm on every rank; the
 * handle owns it). NCCL is resolved at run time (dlopen "libnccl.so.2").
 * rsvd_handle_allreduce_sum is stream-ordered; without a communicator it is a
 * no-op (one rank). */
typedef struct rsvd_handle_s *rsvd_handle;
int rsvd_handle_create(int device, rsvd_handle *out);
int rsvd_handle_destroy(rsvd_handle h);
int rsvd_handle_device(rsvd_handle h, int *device);
int rsvd_handle_world(rsvd_handle h, int *world, int *rank);
int rsvd_handle_set_comm(rsvd_handle h, void *nccl_comm, int world, int rank);
int rsvd_nccl_unique_id(char *id_out, int64_t id_bytes);
int rsvd_handle_init_comm(rsvd_handle h, const char *id, int64_t id_bytes, int world, int rank);
int rsvd_handle_allreduce_sum(rsvd_handle h, void *buf, int64_t count, int dtype, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* RSVD_B200_H */
