// extern "C" entry points (include/rsvd_b200.h): argument validation and
// kernel dispatch. No entry point synchronises the stream.
#include "common.cuh"
#include "gemm.cuh"
#include <stdlib.h>

namespace rsvd {
// small_dense.cu
int64_t chol_deflate_ws_bytes(int64_t p);
int chol_deflate(int64_t p, const double* G, int64_t ldg, const double* ref2, double tau2,
                 double* T, int64_t ldt, int32_t* mask, int32_t* ndef, int32_t* running,
                 const int32_t* active, void* ws, int64_t ws_bytes, const int32_t* pred, cudaStream_t st);
int mask_cols(int dtype, int64_t n, int64_t p, void* X, int64_t ldx, const int32_t* keep,
              const int32_t* pred, cudaStream_t st);
int64_t jacobi_ws_bytes(int64_t n);
int jacobi_sweeps(int64_t n, double* M, int64_t ldm, double* V, int64_t ldv, double tol,
                  int max_sweeps, int32_t* info, double* off_out, void* ws, int64_t ws_bytes,
                  cudaStream_t st);
int eig_select(int64_t w, const double* M, int64_t ldm, const double* V, int64_t ldv, int64_t k,
               double* evals, double* evecs, int64_t lde, void* order_ws, cudaStream_t st);
// syev.cu
int64_t syev_topk_ws_bytes(int64_t w, int64_t k);
int syev_topk(int64_t w, const double* M, int64_t ldm, int64_t k, double* evals, double* evecs, int64_t lde,
              int32_t* info, void* ws, int64_t ws_bytes, cudaStream_t st);
// elementwise.cu
int64_t colreduce_ws_bytes(int64_t n, int64_t p);
int colreduce(int dtype, int square, int64_t n, int64_t p, const void* X, int64_t ldx,
              double* out, void* ws, int64_t ws_bytes, cudaStream_t st);
int canonicalize_signs(int dtype, int64_t n, int64_t k, void* X, int64_t ldx, void* ws,
                       int64_t ws_bytes, cudaStream_t st);
int convert(int sd, int dd, int64_t rows, int64_t cols, const void* src, int64_t lds, void* dst,
            int64_t ldd, const int32_t* pred, cudaStream_t st);
int sqrt_clip(int64_t k, const double* in, double* out, cudaStream_t st);
int move_rows(int dtype, int gather, int64_t nidx, int64_t cols, const int64_t* idx, const void* src, int64_t lds,
              void* dst, int64_t ldd, cudaStream_t st);
int col_absargmax(int dtype, int64_t n, int64_t k, const void* X, int64_t ldx, int64_t row_offset,
                  double* out_val, int64_t* out_idx, void* ws, int64_t ws_bytes, cudaStream_t st);
int flip_by_sign(int dtype, int64_t n, int64_t k, void* X, int64_t ldx, const double* sign_val,
                 cudaStream_t st);
int ortho_error(int64_t k, const double* G, int64_t ldg, double* out, cudaStream_t st);
int insert_fill(int dtype, int64_t n, int64_t p, void* X, int64_t ldx, const int32_t* mask,
                const int32_t* ndef, uint64_t seed, int64_t row_offset, int64_t n_total,
                const int32_t* pred, cudaStream_t st);
int fill_stream(int64_t n, int64_t nvec, uint64_t seed, double* out, cudaStream_t st);
// sparse.cu
int spmm_csr(int dtype, int idx64, int64_t nrows, int64_t ncols, int64_t nb, const void* indptr,
             const void* col, const void* val, const void* B, int64_t ldb, double alpha,
             double beta, void* C, int64_t ldc, cudaStream_t st);
int spmm_nnz_plan(int64_t nnz, int chunk, int64_t nb, const int32_t* col, const float* val, const int32_t* rowid,
                  const float* B, int64_t ldb, double alpha, double beta, float* C, int64_t ldc,
                  const int32_t* head_slot, const int32_t* tail_slot, int64_t nsplit, const int32_t* srow,
                  const int64_t* sbeg, int64_t nempty, const int32_t* empty_rows, float* ws, cudaStream_t st);
int spmm_slab(int64_t nrows, int64_t nb, const int32_t* mptr, const int32_t* midx, const float* mval,
              const int64_t* slab_cols, int64_t M, const float* X, int64_t ldx, float* C, int64_t ldc,
              cudaStream_t st);
int spmm_csr_plan(int dtype, int idx64, int64_t nb, const void* col, const void* val, const void* B, int64_t ldb,
                  double alpha, double beta, void* C, int64_t ldc, int64_t nchunks, const int64_t* clo,
                  const int64_t* chi, const int32_t* crow, const int32_t* cslot, int64_t nsplit,
                  const int32_t* srow, const int64_t* sbeg, void* ws, cudaStream_t st);
int csr_transpose(int dtype, int idx64, int64_t nrows, int64_t ncols, int64_t nnz,
                  const void* indptr, const void* col, const void* val, const int64_t* perm,
                  void* tptr, void* tcol, void* tval, cudaStream_t st);
}  // namespace rsvd

using namespace rsvd;

static bool valid_dtype(int d) { return d == RSVD_F32 || d == RSVD_F64; }

// FP64 products default to the DMMA kernels; RSVD_DISABLE_DMMA=1 selects the
// CUDA-core FP64 kernels (A/B measurement switch).
static bool dmma_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("RSVD_DISABLE_DMMA");
        on = (e && e[0] == '1') ? 0 : 1;
    }
    return on == 1;
}

extern "C" {

int rsvd_gemm_nn(int dtype, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
                 int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc,
                 const double* row_sub, int algo, const int32_t* pred, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype), "gemm_nn: bad dtype %d", dtype);
    RSVD_REQUIRE(m >= 0 && n >= 0 && k >= 0, "gemm_nn: negative dimension");
    RSVD_REQUIRE(lda >= k && ldb >= n && ldc >= n, "gemm_nn: leading dimension too small");
    cudaStream_t st = as_stream(stream);
    if (algo == RSVD_GEMM_SKINNY ||
        (algo == RSVD_GEMM_AUTO && dtype == RSVD_F32 && gemm_skinny_nn_supported(n, k))) {
        RSVD_REQUIRE(dtype == RSVD_F32 && n <= 64, "gemm_nn: skinny path is FP32 with n <= 64");
        return gemm_nn_skinny(m, n, k, alpha, (const float*)A, lda, (const float*)B, ldb, beta,
                              (float*)C, ldc, row_sub, pred, st);
    }
    if (algo == RSVD_GEMM_TC_3XTF32 || (algo == RSVD_GEMM_AUTO && dtype == RSVD_F32 &&
                                         gemm_tc_nn_supported(m, n, k, lda, ldb, ldc, A, B))) {
        RSVD_REQUIRE(dtype == RSVD_F32, "gemm_nn: 3xTF32 path is FP32 only");
        RSVD_REQUIRE(gemm_tc_nn_supported(m, n, k, lda, ldb, ldc, A, B),
                     "gemm_nn: shape/alignment not supported by the tcgen05 kernel");
        return gemm_nn_tc(m, n, k, alpha, (const float*)A, lda, (const float*)B, ldb, beta,
                          (float*)C, ldc, row_sub, pred, st);
    }
    if (algo == RSVD_GEMM_DMMA || (algo == RSVD_GEMM_AUTO && dtype == RSVD_F64 && dmma_enabled())) {
        RSVD_REQUIRE(dtype == RSVD_F64, "gemm_nn: DMMA path is FP64 only");
        return gemm_nn_dmma(m, n, k, alpha, (const double*)A, lda, (const double*)B, ldb, beta,
                            (double*)C, ldc, row_sub, pred, st);
    }
    return gemm_nn_simt(dtype, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, row_sub, pred, st);
}

int64_t rsvd_oz_planes_bytes(int64_t n, int64_t d) { return (n < 0 || d < 0) ? 0 : oz_planes_bytes(n, d); }

int rsvd_oz_num_planes(void) { return oz_num_planes(); }

int rsvd_oz_prepare(int64_t n, int64_t d, const float* A, int64_t lda, int8_t* planes, int32_t* row_exp,
                    void* stream) {
    RSVD_REQUIRE(n >= 0 && d >= 0, "oz_prepare: negative dimension");
    RSVD_REQUIRE(lda >= d, "oz_prepare: leading dimension too small");
    RSVD_REQUIRE(n == 0 || (A && planes && row_exp), "oz_prepare: null pointer");
    return oz_prepare(n, d, A, lda, planes, row_exp, as_stream(stream));
}

int rsvd_oz_prepare_rows(int64_t n, int64_t d, int64_t r0, int64_t nr, const float* A, int64_t lda, int8_t* planes,
                         int32_t* row_exp, void* stream) {
    RSVD_REQUIRE(n >= 0 && d >= 0, "oz_prepare_rows: negative dimension");
    RSVD_REQUIRE(lda >= d, "oz_prepare_rows: leading dimension too small");
    RSVD_REQUIRE(n == 0 || (A && planes && row_exp), "oz_prepare_rows: null pointer");
    return oz_prepare_rows(n, d, r0, nr, A, lda, planes, row_exp, as_stream(stream));
}

int64_t rsvd_oz_gemm_ws_bytes(int trans, int64_t n, int64_t d, int64_t p) {
    if (n < 0 || d < 0 || p < 0) return 0;
    return oz_gemm_ws_bytes(trans, n, d, p);
}

int rsvd_oz_gemm(int trans, int64_t n, int64_t d, int64_t p, double alpha, const int8_t* planes,
                 const int32_t* row_exp, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                 void* ws, int64_t ws_bytes, const int32_t* pred, void* stream) {
    RSVD_REQUIRE(trans >= 0 && trans <= 3, "oz_gemm: trans must be 0 / 1 (+2: reduced accuracy)");
    RSVD_REQUIRE(n >= 0 && d >= 0 && p >= 0, "oz_gemm: negative dimension");
    RSVD_REQUIRE(ldb >= p && ldc >= p, "oz_gemm: leading dimension too small");
    return oz_gemm(trans, n, d, p, alpha, planes, row_exp, B, ldb, beta, C, ldc, ws, ws_bytes, pred,
                   as_stream(stream));
}

int rsvd_oz_basis_planes(void) { return oz_basis_planes(); }

int64_t rsvd_oz_basis_bytes(int64_t n, int64_t w) { return (n < 0 || w < 0) ? 0 : oz_basis_bytes(n, w); }

int64_t rsvd_oz_basis_ws_bytes(int64_t ncols) { return ncols < 0 ? 0 : oz_basis_ws_bytes(ncols); }

int rsvd_oz_basis_slice(int64_t n, int64_t w, const double* Q, int64_t ldq, int64_t c0, int64_t ncols,
                        int8_t* planes, int32_t* col_exp, void* ws, int64_t ws_bytes, void* stream) {
    RSVD_REQUIRE(n >= 0 && w >= 0 && ldq >= w, "oz_basis_slice: bad shape");
    RSVD_REQUIRE(n == 0 || (Q && planes && col_exp), "oz_basis_slice: null pointer");
    return oz_basis_slice(n, w, Q, ldq, c0, ncols, planes, col_exp, ws, ws_bytes, as_stream(stream));
}

int rsvd_oz_gemm_planes(int trans, int64_t n, int64_t d, int64_t p, double alpha, const int8_t* planes, int nplanes,
                        int64_t rows_alloc, int64_t cols_alloc, const int32_t* exps, int col_scaled, const double* B,
                        int64_t ldb, double beta, double* C, int64_t ldc, void* ws, int64_t ws_bytes,
                        const int32_t* pred, void* stream) {
    RSVD_REQUIRE(trans == 0 || trans == 1, "oz_gemm: trans must be 0 or 1");
    RSVD_REQUIRE(n >= 0 && d >= 0 && p >= 0, "oz_gemm: negative dimension");
    RSVD_REQUIRE(ldb >= p && ldc >= p, "oz_gemm: leading dimension too small");
    return oz_gemm_planes(trans, n, d, p, alpha, planes, nplanes, rows_alloc, cols_alloc, exps, col_scaled, B, ldb,
                          beta, C, ldc, ws, ws_bytes, pred, as_stream(stream));
}

int64_t rsvd_split_planes_bytes(int64_t K, int64_t N) { return (K < 0 || N < 0) ? 0 : split_planes_bytes(K, N); }

int rsvd_split_planes(int64_t K, int64_t N, const float* B, int64_t ldb, float* planes, int64_t planes_bytes,
                      const int32_t* pred, void* stream) {
    RSVD_REQUIRE(K >= 0 && N >= 0 && ldb >= N, "split_planes: bad shape");
    RSVD_REQUIRE(planes_bytes >= split_planes_bytes(K, N), "split_planes: plane buffer too small");
    return split_planes(K, N, B, ldb, planes, pred, as_stream(stream));
}

int rsvd_gemm_nn_f32_emit(int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda, const float* B,
                          int64_t ldb, double beta, float* C, int64_t ldc, const double* row_sub, float* planes,
                          int64_t planes_bytes, int32_t* emitted, const int32_t* pred, void* stream) {
    RSVD_REQUIRE(m >= 0 && n >= 0 && k >= 0, "gemm_nn_emit: negative dimension");
    RSVD_REQUIRE(lda >= k && ldb >= n && ldc >= n, "gemm_nn_emit: leading dimension too small");
    RSVD_REQUIRE(emitted != nullptr, "gemm_nn_emit: null pointer");
    cudaStream_t st = as_stream(stream);
    *emitted = 0;
    // planes come out of the tcgen05 kernel's epilogue; any other path computes C only
    if (planes != nullptr && !gemm_skinny_nn_supported(n, k) && gemm_tc_nn_supported(m, n, k, lda, ldb, ldc, A, B)) {
        RSVD_REQUIRE(planes_bytes >= split_planes_bytes(m, n), "gemm_nn_emit: plane buffer too small");
        *emitted = 1;
        return gemm_nn_tc(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, row_sub, pred, st, planes);
    }
    return rsvd_gemm_nn(RSVD_F32, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, row_sub, RSVD_GEMM_AUTO, pred, stream);
}

int rsvd_gemm_tn_f32_planes(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha, const float* A,
                            int64_t lda, const float* B_planes, int64_t planes_bytes, double beta, void* C,
                            int64_t ldc, const double* mu, const double* colsum_b, void* ws, int64_t ws_bytes,
                            const int32_t* pred, void* stream) {
    RSVD_REQUIRE(valid_dtype(out_dtype), "gemm_tn_planes: bad dtype");
    RSVD_REQUIRE(m >= 0 && n >= 0 && k >= 0 && lda >= k && ldc >= n, "gemm_tn_planes: bad shape");
    RSVD_REQUIRE((mu == nullptr) == (colsum_b == nullptr), "gemm_tn_planes: mu and colsum_b go together");
    RSVD_REQUIRE(B_planes != nullptr && planes_bytes >= split_planes_bytes(m, n), "gemm_tn_planes: plane buffer");
    RSVD_REQUIRE(gemm_tc_tn_supported(m, n, k, lda, n, A, B_planes),
                 "gemm_tn_planes: shape/alignment not supported by the tcgen05 kernel");
    return gemm_tn_tc(out_dtype, m, n, k, alpha, A, lda, nullptr, n, beta, C, ldc, mu, colsum_b, ws, ws_bytes, pred,
                      as_stream(stream), B_planes);
}

int rsvd_gemm_tn_f32_planes_ok(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda) {
    return (!gemm_skinny_tn_supported(n, k) && gemm_tc_tn_supported(m, n, k, lda, n, A, A)) ? 1 : 0;
}

int64_t rsvd_gemm_tn_ws_bytes(int dtype, int64_t m, int64_t n, int64_t k, int algo) {
    int64_t a = gemm_tn_simt_ws_bytes(m, n, k);
    if (dtype == RSVD_F64 && algo != RSVD_GEMM_SIMT) {
        int64_t b = gemm_tn_dmma_ws_bytes(m, n, k);
        if (b > a) a = b;
    }
    if (dtype == RSVD_F32 && algo != RSVD_GEMM_SIMT) {
        int64_t b = gemm_tn_tc_ws_bytes(m, n, k);
        if (b > a) a = b;
        if (n <= 64) {
            b = gemm_tn_skinny_ws_bytes(m, n, k);
            if (b > a) a = b;
        }
    }
    return a + 256;
}

int rsvd_gemm_tn(int dtype, int out_dtype, int64_t m, int64_t n, int64_t k, double alpha,
                 const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                 int64_t ldc, const double* mu, const double* colsum_b, void* ws,
                 int64_t ws_bytes, int algo, const int32_t* pred, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype) && valid_dtype(out_dtype), "gemm_tn: bad dtype");
    RSVD_REQUIRE(m >= 0 && n >= 0 && k >= 0, "gemm_tn: negative dimension");
    RSVD_REQUIRE(lda >= k && ldb >= n && ldc >= n, "gemm_tn: leading dimension too small");
    RSVD_REQUIRE((mu == nullptr) == (colsum_b == nullptr), "gemm_tn: mu and colsum_b go together");
    cudaStream_t st = as_stream(stream);
    if (algo == RSVD_GEMM_SKINNY ||
        (algo == RSVD_GEMM_AUTO && dtype == RSVD_F32 && gemm_skinny_tn_supported(n, k))) {
        RSVD_REQUIRE(dtype == RSVD_F32 && n <= 64, "gemm_tn: skinny path is FP32 with n <= 64");
        return gemm_tn_skinny(out_dtype, m, n, k, alpha, (const float*)A, lda, (const float*)B, ldb,
                              beta, C, ldc, mu, colsum_b, ws, ws_bytes, pred, st);
    }
    if (algo == RSVD_GEMM_TC_3XTF32 ||
        (algo == RSVD_GEMM_AUTO && dtype == RSVD_F32 && gemm_tc_tn_supported(m, n, k, lda, ldb, A, B))) {
        RSVD_REQUIRE(dtype == RSVD_F32, "gemm_tn: 3xTF32 path is FP32 only");
        RSVD_REQUIRE(gemm_tc_tn_supported(m, n, k, lda, ldb, A, B),
                     "gemm_tn: shape/alignment not supported by the tcgen05 kernel");
        return gemm_tn_tc(out_dtype, m, n, k, alpha, (const float*)A, lda, (const float*)B, ldb,
                          beta, C, ldc, mu, colsum_b, ws, ws_bytes, pred, st);
    }
    if (algo == RSVD_GEMM_DMMA || (algo == RSVD_GEMM_AUTO && dtype == RSVD_F64 && dmma_enabled())) {
        RSVD_REQUIRE(dtype == RSVD_F64, "gemm_tn: DMMA path is FP64 only");
        return gemm_tn_dmma(out_dtype, m, n, k, alpha, (const double*)A, lda, (const double*)B, ldb,
                            beta, C, ldc, mu, colsum_b, ws, ws_bytes, pred, st);
    }
    return gemm_tn_simt(dtype, out_dtype, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, mu,
                        colsum_b, ws, ws_bytes, pred, st);
}

int rsvd_spmm_csr(int dtype, int idx64, int64_t nrows, int64_t ncols, int64_t nb,
                  const void* indptr, const void* col, const void* val, const void* B,
                  int64_t ldb, double alpha, double beta, void* C, int64_t ldc, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype), "spmm: bad dtype");
    RSVD_REQUIRE(nrows >= 0 && ncols >= 0 && nb >= 0 && ldb >= nb && ldc >= nb, "spmm: bad shape");
    return spmm_csr(dtype, idx64, nrows, ncols, nb, indptr, col, val, B, ldb, alpha, beta, C, ldc,
                    as_stream(stream));
}

int rsvd_spmm_nnz_plan(int64_t nnz, int chunk, int64_t nb, const int32_t* col, const float* val,
                       const int32_t* rowid, const float* B, int64_t ldb, double alpha, double beta, float* C,
                       int64_t ldc, const int32_t* head_slot, const int32_t* tail_slot, int64_t nsplit,
                       const int32_t* split_row, const int64_t* split_beg, int64_t nempty,
                       const int32_t* empty_rows, void* ws, int64_t ws_bytes, void* stream) {
    RSVD_REQUIRE(nnz >= 0 && nb >= 0 && nsplit >= 0 && nempty >= 0, "spmm_nnz_plan: negative size");
    RSVD_REQUIRE(ldb >= nb && ldc >= nb, "spmm_nnz_plan: leading dimension too small");
    RSVD_REQUIRE(nsplit == 0 || (ws && split_row && split_beg), "spmm_nnz_plan: null pointer");
    (void)ws_bytes;
    return spmm_nnz_plan(nnz, chunk, nb, col, val, rowid, B, ldb, alpha, beta, C, ldc, head_slot, tail_slot, nsplit,
                         split_row, split_beg, nempty, empty_rows, (float*)ws, as_stream(stream));
}

int rsvd_spmm_slab(int64_t nrows, int64_t nb, const int32_t* slab_ptr, const int32_t* slab_idx,
                   const float* slab_val, const int64_t* slab_cols, int64_t nslab, const float* X, int64_t ldx,
                   float* C, int64_t ldc, void* stream) {
    RSVD_REQUIRE(nrows >= 0 && nb >= 0 && nslab >= 0, "spmm_slab: negative dimension");
    RSVD_REQUIRE(ldx >= nb && ldc >= nb, "spmm_slab: leading dimension too small");
    RSVD_REQUIRE(nslab * 4 <= 200 * 1024, "spmm_slab: at most 51200 slab columns");
    RSVD_REQUIRE(nrows == 0 || nslab == 0 || (slab_ptr && slab_idx && slab_val && slab_cols && X && C),
                 "spmm_slab: null pointer");
    return spmm_slab(nrows, nb, slab_ptr, slab_idx, slab_val, slab_cols, nslab, X, ldx, C, ldc, as_stream(stream));
}

int rsvd_spmm_csr_plan(int dtype, int idx64, int64_t nrows, int64_t nb, const void* col, const void* val,
                       const void* B, int64_t ldb, double alpha, double beta, void* C, int64_t ldc,
                       int64_t nchunks, const int64_t* chunk_lo, const int64_t* chunk_hi,
                       const int32_t* chunk_row, const int32_t* chunk_slot, int64_t nsplit,
                       const int32_t* split_row, const int64_t* split_beg, void* ws, int64_t ws_bytes,
                       void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype), "spmm_plan: bad dtype");
    RSVD_REQUIRE(nrows >= 0 && nb >= 0 && ldb >= nb && ldc >= nb && nchunks >= 0 && nsplit >= 0,
                 "spmm_plan: bad shape");
    RSVD_REQUIRE(nsplit == 0 || (ws != nullptr && ws_bytes > 0), "spmm_plan: split rows need a workspace");
    (void)nrows;
    return spmm_csr_plan(dtype, idx64, nb, col, val, B, ldb, alpha, beta, C, ldc, nchunks, chunk_lo, chunk_hi,
                         chunk_row, chunk_slot, nsplit, split_row, split_beg, ws, as_stream(stream));
}

int rsvd_csr_transpose(int dtype, int idx64, int64_t nrows, int64_t ncols, int64_t nnz,
                       const void* indptr, const void* col, const void* val,
                       const int64_t* perm_by_col, void* t_indptr, void* t_col, void* t_val,
                       void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype), "csr_transpose: bad dtype");
    RSVD_REQUIRE(nrows >= 0 && ncols >= 0 && nnz >= 0, "csr_transpose: bad shape");
    return csr_transpose(dtype, idx64, nrows, ncols, nnz, indptr, col, val, perm_by_col, t_indptr,
                         t_col, t_val, as_stream(stream));
}

int64_t rsvd_chol_deflate_ws_bytes(int64_t p) { return chol_deflate_ws_bytes(p); }

int rsvd_chol_deflate(int64_t p, const double* G, int64_t ldg, const double* ref2, double tau2,
                      double* Tinv, int64_t ldt, int32_t* mask, int32_t* ndef, int32_t* running,
                      const int32_t* active, void* ws, int64_t ws_bytes, const int32_t* pred,
                      void* stream) {
    RSVD_REQUIRE(p >= 0 && ldg >= p && ldt >= p, "chol_deflate: bad shape");
    return chol_deflate(p, G, ldg, ref2, tau2, Tinv, ldt, mask, ndef, running, active, ws, ws_bytes,
                        pred, as_stream(stream));
}

int rsvd_mask_cols(int dtype, int64_t n, int64_t p, void* X, int64_t ldx, const int32_t* keep,
                   const int32_t* pred, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype) && ldx >= p, "mask_cols: bad args");
    return mask_cols(dtype, n, p, X, ldx, keep, pred, as_stream(stream));
}

int rsvd_insert_fill(int dtype, int64_t n, int64_t p, void* X, int64_t ldx, const int32_t* mask,
                     const int32_t* ndef, uint64_t seed, int64_t row_offset, int64_t n_total,
                     const int32_t* pred, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype) && ldx >= p, "insert_fill: bad args");
    RSVD_REQUIRE(row_offset >= 0 && n_total >= row_offset + n, "insert_fill: bad row range");
    return insert_fill(dtype, n, p, X, ldx, mask, ndef, seed, row_offset, n_total, pred,
                       as_stream(stream));
}

int rsvd_fill_stream(int64_t n, int64_t nvec, uint64_t seed, double* out, void* stream) {
    RSVD_REQUIRE(n >= 0 && nvec >= 0, "fill_stream: bad shape");
    return fill_stream(n, nvec, seed, out, as_stream(stream));
}

int64_t rsvd_jacobi_ws_bytes(int64_t n) { return jacobi_ws_bytes(n); }

int rsvd_jacobi_sweeps(int64_t n, double* M, int64_t ldm, double* V, int64_t ldv, double tol,
                       int max_sweeps, int32_t* info, double* off_out, void* ws, int64_t ws_bytes,
                       void* stream) {
    RSVD_REQUIRE(n >= 1 && ldm >= n && ldv >= n, "jacobi: bad shape");
    RSVD_REQUIRE(tol >= 0.0 && max_sweeps >= 0, "jacobi: bad tol/max_sweeps");
    return jacobi_sweeps(n, M, ldm, V, ldv, tol, max_sweeps, info, off_out, ws, ws_bytes,
                         as_stream(stream));
}

int rsvd_eig_select(int64_t w, const double* M, int64_t ldm, const double* V, int64_t ldv,
                    int64_t k, double* evals, double* evecs, int64_t lde, int32_t* order_ws,
                    void* stream) {
    RSVD_REQUIRE(w >= 1 && k >= 0 && k <= w && lde >= k, "eig_select: bad shape");
    return eig_select(w, M, ldm, V, ldv, k, evals, evecs, lde, order_ws, as_stream(stream));
}

int64_t rsvd_syev_topk_ws_bytes(int64_t w, int64_t k) { return syev_topk_ws_bytes(w, k); }

int rsvd_syev_topk(int64_t w, const double* M, int64_t ldm, int64_t k, double* evals, double* evecs,
                   int64_t lde, int32_t* info, void* ws, int64_t ws_bytes, void* stream) {
    RSVD_REQUIRE(w >= 1 && k >= 1 && k <= w && ldm >= w && lde >= k, "syev_topk: bad shape");
    return syev_topk(w, M, ldm, k, evals, evecs, lde, info, ws, ws_bytes, as_stream(stream));
}

int64_t rsvd_colreduce_ws_bytes(int64_t n, int64_t p) { return colreduce_ws_bytes(n, p); }

int rsvd_colreduce(int dtype, int square, int64_t n, int64_t p, const void* X, int64_t ldx,
                   double* out, void* ws, int64_t ws_bytes, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype) && ldx >= p, "colreduce: bad args");
    return colreduce(dtype, square, n, p, X, ldx, out, ws, ws_bytes, as_stream(stream));
}

int rsvd_canonicalize_signs(int dtype, int64_t n, int64_t k, void* X, int64_t ldx, void* ws,
                            int64_t ws_bytes, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype) && ldx >= k, "canonicalize_signs: bad args");
    return canonicalize_signs(dtype, n, k, X, ldx, ws, ws_bytes, as_stream(stream));
}

int rsvd_col_absargmax(int dtype, int64_t n, int64_t k, const void* X, int64_t ldx,
                       int64_t row_offset, double* out_val, int64_t* out_idx, void* ws,
                       int64_t ws_bytes, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype) && ldx >= k, "col_absargmax: bad args");
    return col_absargmax(dtype, n, k, X, ldx, row_offset, out_val, out_idx, ws, ws_bytes,
                         as_stream(stream));
}

int rsvd_flip_by_sign(int dtype, int64_t n, int64_t k, void* X, int64_t ldx,
                      const double* sign_val, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype) && ldx >= k, "flip_by_sign: bad args");
    return flip_by_sign(dtype, n, k, X, ldx, sign_val, as_stream(stream));
}

int rsvd_convert(int src_dtype, int dst_dtype, int64_t rows, int64_t cols, const void* src,
                 int64_t lds, void* dst, int64_t ldd, const int32_t* pred, void* stream) {
    RSVD_REQUIRE(valid_dtype(src_dtype) && valid_dtype(dst_dtype), "convert: bad dtype");
    RSVD_REQUIRE(lds >= cols && ldd >= cols, "convert: bad leading dimension");
    return convert(src_dtype, dst_dtype, rows, cols, src, lds, dst, ldd, pred, as_stream(stream));
}

int rsvd_gather_rows(int dtype, int64_t nidx, int64_t cols, const int64_t* idx, const void* src, int64_t lds,
                     void* dst, int64_t ldd, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype), "gather_rows: bad dtype");
    RSVD_REQUIRE(nidx >= 0 && cols >= 0 && lds >= cols && ldd >= cols, "gather_rows: bad shape");
    return move_rows(dtype, 1, nidx, cols, idx, src, lds, dst, ldd, as_stream(stream));
}

int rsvd_scatter_rows(int dtype, int64_t nidx, int64_t cols, const int64_t* idx, const void* src, int64_t lds,
                      void* dst, int64_t ldd, void* stream) {
    RSVD_REQUIRE(valid_dtype(dtype), "scatter_rows: bad dtype");
    RSVD_REQUIRE(nidx >= 0 && cols >= 0 && lds >= cols && ldd >= cols, "scatter_rows: bad shape");
    return move_rows(dtype, 0, nidx, cols, idx, src, lds, dst, ldd, as_stream(stream));
}

int rsvd_sqrt_clip(int64_t k, const double* in, double* out, void* stream) {
    return sqrt_clip(k, in, out, as_stream(stream));
}

int rsvd_ortho_error(int64_t k, const double* G, int64_t ldg, double* out, void* stream) {
    RSVD_REQUIRE(k >= 0 && ldg >= k, "ortho_error: bad shape");
    return ortho_error(k, G, ldg, out, as_stream(stream));
}

}  // extern "C"
