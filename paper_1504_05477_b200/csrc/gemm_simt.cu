// CUDA-core tall-skinny products: the FP64 path (oracle-parity precision) and
// the FP32 fallback for shapes the tensor-core kernel does not take.
//
//   gemm_nn:  C = alpha (A B - 1 row_sub^T) + beta C     A m x k, B k x n
//   gemm_tn:  C = alpha (A^T B - mu colsum^T) + beta C   reduction over m,
//             fixed split order, FP64 partials -> deterministic.
//
// Replaces _kernels.pyx:56-71 (mm) as called through MatrixOperator.apply /
// apply_transpose (matrix.py:227-247) and the BLAS-2 projections of _mgs
// (factor.py:93-98).
#include "common.cuh"
#include "gemm.cuh"

namespace rsvd {

namespace {

constexpr int kThreads = 256;

template <typename T, int BM, int BN, int BK>
__global__ void __launch_bounds__(kThreads)
k_gemm_nn(int64_t m, int64_t n, int64_t k, double alpha, const T* __restrict__ A, int64_t lda,
          const T* __restrict__ B, int64_t ldb, double beta, T* __restrict__ C, int64_t ldc,
          const double* __restrict__ row_sub, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    constexpr int TM = BM / 16, TN = BN / 16;
    __shared__ T As[2][BK][BM + 2];
    __shared__ T Bs[2][BK][BN];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

    constexpr int A_PER = BM * BK / kThreads;
    constexpr int B_PER = BK * BN / kThreads;
    T ra[A_PER], rb[B_PER];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int t = 0; t < A_PER; ++t) {
            int idx = threadIdx.x + t * kThreads;
            int r = idx / BK, c = idx % BK;
            int64_t gr = m0 + r, gc = k0 + c;
            ra[t] = (gr < m && gc < k) ? A[gr * lda + gc] : T(0);
        }
#pragma unroll
        for (int t = 0; t < B_PER; ++t) {
            int idx = threadIdx.x + t * kThreads;
            int r = idx / BN, c = idx % BN;
            int64_t gr = k0 + r, gc = n0 + c;
            rb[t] = (gr < k && gc < n) ? B[gr * ldb + gc] : T(0);
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int t = 0; t < A_PER; ++t) {
            int idx = threadIdx.x + t * kThreads;
            As[buf][idx % BK][idx / BK] = ra[t];
        }
#pragma unroll
        for (int t = 0; t < B_PER; ++t) {
            int idx = threadIdx.x + t * kThreads;
            Bs[buf][idx / BN][idx % BN] = rb[t];
        }
    };
    int buf = 0;
    load(0);
    store(0);
    __syncthreads();
    for (int64_t k0 = 0; k0 < k; k0 += BK) {
        const bool more = k0 + BK < k;
        if (more) load(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            T a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < TN; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        if (more) {
            store(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        int64_t r = m0 + ty + 16 * i;
        if (r >= m) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            int64_t c = n0 + tx + 16 * j;
            if (c >= n) continue;
            double v = (double)acc[i][j];
            if (row_sub) v -= row_sub[c];
            v *= alpha;
            if (beta != 0.0) v += beta * (double)C[r * ldc + c];
            C[r * ldc + c] = (T)v;
        }
    }
}

// Partial A^T B over one split of the rows; FP64 accumulation.
template <typename T, int BKO, int BN, int BR>
__global__ void __launch_bounds__(kThreads)
k_gemm_tn_partial(int64_t m, int64_t n, int64_t k, const T* __restrict__ A, int64_t lda,
                  const T* __restrict__ B, int64_t ldb, int64_t rows_per_split,
                  double* __restrict__ ws, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    constexpr int TM = BKO / 16, TN = BN / 16;
    __shared__ T As[2][BR][BKO];
    __shared__ T Bs[2][BR][BN];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t k0 = (int64_t)blockIdx.x * BKO, n0 = (int64_t)blockIdx.y * BN;
    const int64_t s = blockIdx.z;
    const int64_t rbeg = s * rows_per_split;
    const int64_t rend = min(m, rbeg + rows_per_split);
    double acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
    constexpr int A_PER = BR * BKO / kThreads;
    constexpr int B_PER = BR * BN / kThreads;
    T ra[A_PER], rb[B_PER];
    auto load = [&](int64_t r0) {
#pragma unroll
        for (int t = 0; t < A_PER; ++t) {
            int idx = threadIdx.x + t * kThreads;
            int r = idx / BKO, c = idx % BKO;
            int64_t gr = r0 + r, gc = k0 + c;
            ra[t] = (gr < rend && gc < k) ? A[gr * lda + gc] : T(0);
        }
#pragma unroll
        for (int t = 0; t < B_PER; ++t) {
            int idx = threadIdx.x + t * kThreads;
            int r = idx / BN, c = idx % BN;
            int64_t gr = r0 + r, gc = n0 + c;
            rb[t] = (gr < rend && gc < n) ? B[gr * ldb + gc] : T(0);
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int t = 0; t < A_PER; ++t) {
            int idx = threadIdx.x + t * kThreads;
            As[buf][idx / BKO][idx % BKO] = ra[t];
        }
#pragma unroll
        for (int t = 0; t < B_PER; ++t) {
            int idx = threadIdx.x + t * kThreads;
            Bs[buf][idx / BN][idx % BN] = rb[t];
        }
    };
    if (rbeg < rend) {
        int buf = 0;
        load(rbeg);
        store(0);
        __syncthreads();
        for (int64_t r0 = rbeg; r0 < rend; r0 += BR) {
            const bool more = r0 + BR < rend;
            if (more) load(r0 + BR);
#pragma unroll
            for (int rr = 0; rr < BR; ++rr) {
                double a[TM], b[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) a[i] = (double)As[buf][rr][ty + 16 * i];
#pragma unroll
                for (int j = 0; j < TN; ++j) b[j] = (double)Bs[buf][rr][tx + 16 * j];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
            }
            if (more) {
                store(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        int64_t r = k0 + ty + 16 * i;
        if (r >= k) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            int64_t c = n0 + tx + 16 * j;
            if (c >= n) continue;
            ws[(s * k + r) * n + c] = acc[i][j];
        }
    }
}

template <typename TO>
__global__ void k_tn_reduce(int64_t k, int64_t n, int64_t splits, const double* __restrict__ ws,
                            double alpha, double beta, TO* __restrict__ C, int64_t ldc,
                            const double* __restrict__ mu, const double* __restrict__ cs,
                            const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * n) return;
    int64_t r = idx / n, c = idx % n;
    double v = 0.0;
    for (int64_t s = 0; s < splits; ++s) v += ws[s * k * n + idx];
    if (mu) v -= mu[r] * cs[c];
    v *= alpha;
    if (beta != 0.0) v += beta * (double)C[r * ldc + c];
    C[r * ldc + c] = (TO)v;
}

constexpr int TN_BKO = 64, TN_BN = 64, TN_BR = 16;

int64_t tn_splits(int64_t m, int64_t n, int64_t k) {
    int64_t tiles = cdiv(k, TN_BKO) * cdiv(n, TN_BN);
    int64_t target = (int64_t)sm_count() * 4;
    int64_t s = cdiv(target, tiles);
    int64_t max_s = cdiv(m, 1024);
    if (s > max_s) s = max_s;
    if (s < 1) s = 1;
    return s;
}

}  // namespace

int gemm_nn_simt(int dtype, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
                 int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc,
                 const double* row_sub, const int32_t* pred, cudaStream_t st) {
    if (m == 0 || n == 0) return RSVD_OK;
    if (dtype == RSVD_F64) {
        constexpr int BM = 64, BN = 64, BK = 16;
        dim3 grid((unsigned)cdiv(m, BM), (unsigned)cdiv(n, BN));
        k_gemm_nn<double, BM, BN, BK><<<grid, kThreads, 0, st>>>(
            m, n, k, alpha, (const double*)A, lda, (const double*)B, ldb, beta, (double*)C, ldc,
            row_sub, pred);
    } else {
        constexpr int BM = 64, BN = 64, BK = 16;
        dim3 grid((unsigned)cdiv(m, BM), (unsigned)cdiv(n, BN));
        k_gemm_nn<float, BM, BN, BK><<<grid, kThreads, 0, st>>>(
            m, n, k, alpha, (const float*)A, lda, (const float*)B, ldb, beta, (float*)C, ldc,
            row_sub, pred);
    }
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int64_t gemm_tn_simt_ws_bytes(int64_t m, int64_t n, int64_t k) {
    int64_t s = tn_splits(m, n, k);
    return s * k * n * (int64_t)sizeof(double);
}

int gemm_tn_simt(int dtype, int out_dtype, int64_t m, int64_t n, int64_t k, double alpha,
                 const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                 int64_t ldc, const double* mu, const double* cs, void* ws, int64_t ws_bytes,
                 const int32_t* pred, cudaStream_t st) {
    if (k == 0 || n == 0) return RSVD_OK;
    int64_t s = tn_splits(m, n, k);
    RSVD_REQUIRE(ws_bytes >= s * k * n * (int64_t)sizeof(double), "gemm_tn: workspace too small");
    int64_t rps = cdiv(cdiv(m, s), TN_BR) * TN_BR;
    dim3 grid((unsigned)cdiv(k, TN_BKO), (unsigned)cdiv(n, TN_BN), (unsigned)s);
    if (dtype == RSVD_F64)
        k_gemm_tn_partial<double, TN_BKO, TN_BN, TN_BR><<<grid, kThreads, 0, st>>>(
            m, n, k, (const double*)A, lda, (const double*)B, ldb, rps, (double*)ws, pred);
    else
        k_gemm_tn_partial<float, TN_BKO, TN_BN, TN_BR><<<grid, kThreads, 0, st>>>(
            m, n, k, (const float*)A, lda, (const float*)B, ldb, rps, (double*)ws, pred);
    RSVD_CHECK_LAUNCH();
    int64_t tot = k * n;
    unsigned nb = (unsigned)cdiv(tot, 256);
    if (out_dtype == RSVD_F64)
        k_tn_reduce<double><<<nb, 256, 0, st>>>(k, n, s, (const double*)ws, alpha, beta,
                                                (double*)C, ldc, mu, cs, pred);
    else
        k_tn_reduce<float><<<nb, 256, 0, st>>>(k, n, s, (const double*)ws, alpha, beta, (float*)C,
                                               ldc, mu, cs, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace rsvd
