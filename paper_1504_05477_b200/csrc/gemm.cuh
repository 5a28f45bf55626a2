// Internal GEMM entry points (dispatched from api.cu).
#pragma once
#include "common.cuh"

namespace rsvd {

// true when the op must be skipped (device-side predicate, see the header)
__device__ __forceinline__ bool pred_off(const int32_t* pred) { return pred && *pred == 0; }

int gemm_nn_simt(int dtype, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
                 int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc,
                 const double* row_sub, const int32_t* pred, cudaStream_t st);
int64_t gemm_tn_simt_ws_bytes(int64_t m, int64_t n, int64_t k);
int gemm_tn_simt(int dtype, int out_dtype, int64_t m, int64_t n, int64_t k, double alpha,
                 const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                 int64_t ldc, const double* mu, const double* cs, void* ws, int64_t ws_bytes,
                 const int32_t* pred, cudaStream_t st);

// tcgen05 3xTF32 kernels (gemm_tc.cu). Return RSVD_ERR_INVALID when the
// shape/alignment is not supported so the dispatcher can refuse loudly.
bool gemm_tc_nn_supported(int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb,
                          int64_t ldc, const void* A, const void* B);
int gemm_nn_tc(int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda,
               const float* B, int64_t ldb, double beta, float* C, int64_t ldc,
               const double* row_sub, const int32_t* pred, cudaStream_t st, float* emit = nullptr);
int64_t split_planes_bytes(int64_t K, int64_t N);
int split_planes(int64_t K, int64_t N, const float* B, int64_t ldb, float* planes, const int32_t* pred,
                 cudaStream_t st);
bool gemm_tc_tn_supported(int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb,
                          const void* A, const void* B);
int64_t gemm_tn_tc_ws_bytes(int64_t m, int64_t n, int64_t k);
int gemm_tn_tc(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha, const float* A,
               int64_t lda, const float* B, int64_t ldb, double beta, void* C, int64_t ldc,
               const double* mu, const double* cs, void* ws, int64_t ws_bytes, const int32_t* pred,
               cudaStream_t st, const float* b_planes = nullptr);

// FP64 tensor-core (mma.sync f64) kernels (gemm_dmma.cu).
int gemm_nn_dmma(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                 const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                 const double* row_sub, const int32_t* pred, cudaStream_t st);
int64_t gemm_tn_dmma_ws_bytes(int64_t m, int64_t n, int64_t k);
int gemm_tn_dmma(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                 int64_t lda, const double* B, int64_t ldb, double beta, void* C, int64_t ldc,
                 const double* mu, const double* cs, void* ws, int64_t ws_bytes, const int32_t* pred,
                 cudaStream_t st);

// FP32 CUDA-core kernels for outputs <= 64 columns wide (skinny.cu).
bool gemm_skinny_nn_supported(int64_t n, int64_t k);
bool gemm_skinny_tn_supported(int64_t n, int64_t k);
int gemm_nn_skinny(int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda,
                   const float* B, int64_t ldb, double beta, float* C, int64_t ldc,
                   const double* row_sub, const int32_t* pred, cudaStream_t st);
int64_t gemm_tn_skinny_ws_bytes(int64_t m, int64_t n, int64_t k);
int gemm_tn_skinny(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha, const float* A,
                   int64_t lda, const float* B, int64_t ldb, double beta, void* C, int64_t ldc,
                   const double* mu, const double* cs, void* ws, int64_t ws_bytes,
                   const int32_t* pred, cudaStream_t st);

// int8 Ozaki FP64-accurate products of an FP32 A (gemm_oz.cu).
int64_t oz_planes_bytes(int64_t n, int64_t d);
int oz_num_planes();
int oz_prepare(int64_t n, int64_t d, const float* A, int64_t lda, int8_t* planes, int32_t* row_exp,
               cudaStream_t st);
int oz_prepare_rows(int64_t n, int64_t d, int64_t r0, int64_t nr, const float* A, int64_t lda, int8_t* planes,
                    int32_t* row_exp, cudaStream_t st);
int64_t oz_gemm_ws_bytes(int trans, int64_t n, int64_t d, int64_t p);
int oz_gemm_planes(int trans, int64_t n, int64_t d, int64_t p, double alpha, const int8_t* planes, int nplanes,
                   int64_t rows_alloc, int64_t cols_alloc, const int32_t* exps, int col_scaled, const double* B,
                   int64_t ldb, double beta, double* C, int64_t ldc, void* ws, int64_t ws_bytes, const int32_t* pred,
                   cudaStream_t st, int reduced = 0);
int oz_basis_planes();
int64_t oz_basis_bytes(int64_t n, int64_t w);
int64_t oz_basis_ws_bytes(int64_t ncols);
int oz_basis_slice(int64_t n, int64_t w, const double* Q, int64_t ldq, int64_t c0, int64_t ncols, int8_t* planes,
                   int32_t* col_exp, void* ws, int64_t ws_bytes, cudaStream_t st);
int oz_gemm(int trans, int64_t n, int64_t d, int64_t p, double alpha, const int8_t* planes,
            const int32_t* row_exp, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* ws,
            int64_t ws_bytes, const int32_t* pred, cudaStream_t st);

}  // namespace rsvd
