// FP32 CUDA-core kernels for the orthonormalization-sized products, where the
// output is at most 64 columns wide and the inner dimension of NN is small:
//   NN  C[m x n] = alpha (A[m x k] B[k x n] - 1 row_sub^T) + beta C
//       (V R^{-1} of a CholeskyQR step, k = p; V -= Q c projections)
//   TN  C[k x n] = alpha (A^T B - mu colsum^T) + beta C, A m x k, B m x n
//       (block Grams V^T V and projection coefficients Q^T V, k <= ~1000)
// These products move ~10-100 MB and do little arithmetic; the tcgen05
// kernel's per-CTA fixed cost (TMEM allocation, 11 warp roles, drain
// epilogue) and its B pre-split dominate them, so they get lean one-pass
// kernels instead. Arithmetic: FP32 FMAs, TN folds every 32-row chunk into
// FP64 accumulators and writes FP64 split partials that k_skinny_reduce sums
// in a fixed order (deterministic, no atomics).
#include "gemm.cuh"
#include <stdlib.h>

namespace rsvd {

namespace {

constexpr int kSkThreads = 256;
constexpr int kNnThreads = 128;
constexpr int kNnRows = 64;  // NN rows per CTA
constexpr int kKc = 32;      // inner-dimension chunk

// NN: 128 threads = 8 (x) x 16 (y); thread (tx, ty) owns rows 4 ty .. 4 ty + 3
// and columns 8 tx .. 8 tx + 7. A chunk is row-major in smem with a 33-float
// pitch (conflict-free stores and reads); the next k-chunk is prefetched
// into registers while the current one is multiplied.
__global__ void __launch_bounds__(kNnThreads, 4)
k_skinny_nn(int64_t m, int n, int k, double alpha, const float* __restrict__ A, int64_t lda,
            const float* __restrict__ B, int64_t ldb, double beta, float* __restrict__ C, int64_t ldc,
            const double* __restrict__ row_sub, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    __shared__ float As[kNnRows][kKc + 1];
    __shared__ __align__(16) float Bs[kKc][64];
    const int t = threadIdx.x, tx = t % 8, ty = t / 8;
    const int64_t r0 = (int64_t)blockIdx.x * kNnRows;
    constexpr int LA = kNnRows * kKc / kNnThreads;  // 16: rows 4 i + t / 32, k = t % 32
    constexpr int LB = kKc * 64 / kNnThreads;       // 16: k = (i * 128 + t) / 64, column t % 64
    float ra[LA], rb[LB];
    const int kl = t % 32, wr = t / 32, cb = t % 64, kb = t / 64;
    auto load = [&](int k0) {
#pragma unroll
        for (int i = 0; i < LA; ++i) {
            const int64_t row = r0 + 4 * i + wr;
            ra[i] = (row < m && k0 + kl < k) ? A[row * lda + k0 + kl] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int kk = 2 * i + kb;
            rb[i] = (k0 + kk < k && cb < n) ? B[(int64_t)(k0 + kk) * ldb + cb] : 0.f;
        }
    };
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    load(0);
    for (int k0 = 0; k0 < k; k0 += kKc) {
#pragma unroll
        for (int i = 0; i < LA; ++i) As[4 * i + wr][kl] = ra[i];
#pragma unroll
        for (int i = 0; i < LB; ++i) Bs[2 * i + kb][cb] = rb[i];
        __syncthreads();
        if (k0 + kKc < k) load(k0 + kKc);
        const int kn = min(kKc, k - k0);
        for (int kk = 0; kk < kn; ++kk) {
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][8 * tx]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[kk][8 * tx + 4]);
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float a = As[4 * ty + i][kk];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a, bv[j], acc[i][j]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t row = r0 + 4 * ty + i;
        if (row >= m) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = 8 * tx + j;
            if (c >= n) continue;
            double r = (double)acc[i][j];
            if (row_sub) r -= row_sub[c];
            r *= alpha;
            if (beta != 0.0) r += beta * (double)C[row * ldc + c];
            C[row * ldc + c] = (float)r;
        }
    }
}

// NN (v2): 256 threads, 128 rows per CTA. The CTA stages B (k x 64, zero
// columns past n) and its 128 x k slab of A in shared memory (16-byte loads
// when A's rows are 16-byte aligned, as rows_buffer guarantees; pitch k + 1
// so the 4 rows a warp reads per step fall in distinct banks); thread
// (tx, ty) owns rows 4 ty .. 4 ty + 3 and columns 8 tx .. 8 tx + 7. The
// results go back through shared memory so the epilogue (row_sub, alpha,
// beta C) reads and writes C row-contiguously.
constexpr int kNn2Threads = 256, kNn2Rows = 128, kNn2CPitch = 65;

__host__ __device__ constexpr int nn2_a_floats(int k) {
    return kNn2Rows * (k + 1) > kNn2Rows * kNn2CPitch ? kNn2Rows * (k + 1) : kNn2Rows * kNn2CPitch;
}

template <bool VEC>
__global__ void __launch_bounds__(kNn2Threads, 3)
k_skinny_nn2(int64_t m, int n, int k, double alpha, const float* __restrict__ A, int64_t lda,
             const float* __restrict__ B, int64_t ldb, double beta, float* __restrict__ C, int64_t ldc,
             const double* __restrict__ row_sub, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    extern __shared__ __align__(16) float sm2[];
    float* Bs = sm2;              // k x 64
    float* As = sm2 + k * 64;     // 128 x (k + 1), later the 128 x 65 result tile
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * kNn2Rows;
    const int PA = k + 1;
    if (VEC) {
        const int k4 = (k + 3) / 4;
#pragma unroll 4
        for (int idx = t; idx < kNn2Rows * k4; idx += kNn2Threads) {
            const int r = idx / k4, c = 4 * (idx % k4);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r0 + r < m) v = __ldg(reinterpret_cast<const float4*>(A + (r0 + r) * lda + c));
            float* d = As + r * PA + c;
            d[0] = v.x;
            if (c + 1 < k) d[1] = v.y;
            if (c + 2 < k) d[2] = v.z;
            if (c + 3 < k) d[3] = v.w;
        }
    } else {
#pragma unroll 4
        for (int idx = t; idx < kNn2Rows * k; idx += kNn2Threads) {
            const int r = idx / k, c = idx % k;
            As[r * PA + c] = (r0 + r < m) ? __ldg(A + (r0 + r) * lda + c) : 0.f;
        }
    }
    for (int idx = t; idx < k * 64; idx += kNn2Threads) {
        const int kk = idx / 64, c = idx % 64;
        Bs[idx] = c < n ? __ldg(B + (int64_t)kk * ldb + c) : 0.f;
    }
    __syncthreads();
    const int tx = t % 8, ty = t / 8;
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    const float* a_row = As + 4 * ty * PA;
#pragma unroll 2
    for (int kk = 0; kk < k; ++kk) {
        const float4 b0 = *reinterpret_cast<const float4*>(Bs + kk * 64 + 8 * tx);
        const float4 b1 = *reinterpret_cast<const float4*>(Bs + kk * 64 + 8 * tx + 4);
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float a = a_row[i * PA + kk];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a, bv[j], acc[i][j]);
        }
    }
    __syncthreads();  // As is reused for the result tile
    float* Cs = As;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) Cs[(4 * ty + i) * kNn2CPitch + 8 * tx + j] = acc[i][j];
    __syncthreads();
    const int rows = (int)min((int64_t)kNn2Rows, m - r0);
    for (int idx = t; idx < rows * n; idx += kNn2Threads) {
        const int r = idx / n, c = idx % n;
        double v = (double)Cs[r * kNn2CPitch + c];
        if (row_sub) v -= row_sub[c];
        v *= alpha;
        float* out = C + (r0 + r) * ldc + c;
        if (beta != 0.0) v += beta * (double)*out;
        *out = (float)v;
    }
}

// TN partial: CTA (x = split, y = 64-wide tile of A's columns) reduces rows
// [x rps, (x+1) rps) into a 64 x 64 block; thread (tx, ty) owns outputs
// (4 ty + i, 4 tx + j). Chunks of 32 rows are multiplied in FP32 and folded
// into FP64 accumulators; the next chunk is prefetched into registers.
__global__ void __launch_bounds__(kSkThreads, 2)
k_skinny_tn(int64_t m, int k, int n, const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
            int64_t ldb, int64_t rps, double* __restrict__ ws, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    __shared__ __align__(16) float As[kKc][64 + 4];
    __shared__ __align__(16) float Bs[kKc][64 + 4];
    const int t = threadIdx.x, tx = t % 16, ty = t / 16;
    const int c0 = blockIdx.y * 64;
    const int64_t rbeg = (int64_t)blockIdx.x * rps, rend = min(m, rbeg + rps);
    constexpr int L = kKc * 64 / kSkThreads;  // 8 values of each operand per thread per chunk
    float ra[L], rb[L];
    const int c = t % 64;
    const bool a_ok = c0 + c < k, b_ok = c < n;
    auto load = [&](int64_t q0) {
#pragma unroll
        for (int i = 0; i < L; ++i) {
            const int64_t row = q0 + i * (kSkThreads / 64) + t / 64;
            const bool r_ok = row < rend;
            ra[i] = (r_ok && a_ok) ? A[row * lda + c0 + c] : 0.f;
            rb[i] = (r_ok && b_ok) ? B[row * ldb + c] : 0.f;
        }
    };
    double dacc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dacc[i][j] = 0.0;
    if (rbeg < rend) load(rbeg);
    for (int64_t q0 = rbeg; q0 < rend; q0 += kKc) {
#pragma unroll
        for (int i = 0; i < L; ++i) {
            As[i * (kSkThreads / 64) + t / 64][c] = ra[i];
            Bs[i * (kSkThreads / 64) + t / 64][c] = rb[i];
        }
        __syncthreads();
        if (q0 + kKc < rend) load(q0 + kKc);
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 8
        for (int kk = 0; kk < kKc; ++kk) {
            const float4 a = *reinterpret_cast<const float4*>(&As[kk][4 * ty]);
            const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][4 * tx]);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dacc[i][j] += (double)acc[i][j];
        __syncthreads();
    }
    double* out = ws + (int64_t)blockIdx.x * k * n;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = c0 + 4 * ty + i;
        if (r >= k) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cc = 4 * tx + j;
            if (cc < n) out[(int64_t)r * n + cc] = dacc[i][j];
        }
    }
}

// Sum of the split partials in a fixed order: block = 32 outputs x 32 split
// groups; group g sums splits g, g + 32, ...; the group sums are added in
// group order. Deterministic for a fixed split count. (8 groups left each
// thread ~33 dependent L2 loads: 10 us for a 50 x 50 Gram over 261 splits.)
constexpr int kRedGroups = 32;  // split groups per 32 outputs (1024 threads)

template <typename TO>
__global__ void __launch_bounds__(32 * kRedGroups)
k_skinny_reduce(int64_t k, int64_t n, int64_t splits, const double* __restrict__ ws, double alpha,
                double beta, TO* __restrict__ C, int64_t ldc, const double* __restrict__ mu,
                const double* __restrict__ cs, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    __shared__ double part[kRedGroups][33];
    const int o = threadIdx.x % 32, g = threadIdx.x / 32;
    const int64_t e = (int64_t)blockIdx.x * 32 + o;
    const int64_t tot = k * n;
    double v = 0.0;
    if (e < tot)
        for (int64_t s = g; s < splits; s += kRedGroups) v += ws[s * tot + e];
    part[g][o] = v;
    __syncthreads();
    if (g != 0 || e >= tot) return;
    double r = part[0][o];
#pragma unroll
    for (int i = 1; i < kRedGroups; ++i) r += part[i][o];
    const int64_t row = e / n, col = e % n;
    if (mu) r -= mu[row] * cs[col];
    r *= alpha;
    if (beta != 0.0) r += beta * (double)C[row * ldc + col];
    C[row * ldc + col] = (TO)r;
}

int64_t tn_splits(int64_t m, int64_t k) {
    const int64_t tiles = cdiv(k, 64);
    int64_t s = cdiv(2 * (int64_t)sm_count(), tiles);
    const int64_t max_s = cdiv(m, 4 * kKc);  // at least 4 chunks per split
    if (s > max_s) s = max_s;
    return s < 1 ? 1 : s;
}

}  // namespace

// measured crossover vs the tcgen05 kernel at n = 50 (tools/bench_small.py):
// NN wins to k ~ 128, TN only for Gram-sized outputs
bool gemm_skinny_nn_supported(int64_t n, int64_t k) { return n <= 64 && k <= 128; }
bool gemm_skinny_tn_supported(int64_t n, int64_t k) { return n <= 64 && k <= 64; }

int gemm_nn_skinny(int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda, const float* B,
                   int64_t ldb, double beta, float* C, int64_t ldc, const double* row_sub, const int32_t* pred,
                   cudaStream_t st) {
    RSVD_REQUIRE(n <= 64, "gemm_nn_skinny: n = %lld > 64", (long long)n);
    if (m == 0 || n == 0) return RSVD_OK;
    if (k > 64) {  // k_skinny_nn2 measured faster at k = 50, slower at k = 100 (47.9 vs 41.4 us)
        k_skinny_nn<<<(unsigned)cdiv(m, kNnRows), kNnThreads, 0, st>>>(m, (int)n, (int)k, alpha, A, lda, B, ldb,
                                                                      beta, C, ldc, row_sub, pred);
        RSVD_CHECK_LAUNCH();
        return RSVD_OK;
    }
    const int kk = k < 1 ? 1 : (int)k;
    const size_t smem = (size_t)(kk * 64 + nn2_a_floats(kk)) * sizeof(float);
    const bool vec = lda % 4 == 0 && ((uintptr_t)A % 16) == 0;
    const unsigned grid = (unsigned)cdiv(m, kNn2Rows);
    if (vec) {
        static PerDevice<bool> attr_dev;
        bool& attr = attr_dev.get();
        if (!attr) {
            RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_skinny_nn2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)(128 * 64 * 4 + nn2_a_floats(128) * 4)));
            attr = true;
        }
        k_skinny_nn2<true><<<grid, kNn2Threads, smem, st>>>(m, (int)n, (int)k, alpha, A, lda, B, ldb, beta, C, ldc,
                                                             row_sub, pred);
    } else {
        static PerDevice<bool> attr_dev;
        bool& attr = attr_dev.get();
        if (!attr) {
            RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_skinny_nn2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)(128 * 64 * 4 + nn2_a_floats(128) * 4)));
            attr = true;
        }
        k_skinny_nn2<false><<<grid, kNn2Threads, smem, st>>>(m, (int)n, (int)k, alpha, A, lda, B, ldb, beta, C,
                                                              ldc, row_sub, pred);
    }
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int64_t gemm_tn_skinny_ws_bytes(int64_t m, int64_t n, int64_t k) {
    return tn_splits(m, k) * k * n * (int64_t)sizeof(double);
}

int gemm_tn_skinny(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda,
                   const float* B, int64_t ldb, double beta, void* C, int64_t ldc, const double* mu,
                   const double* cs, void* ws, int64_t ws_bytes, const int32_t* pred, cudaStream_t st) {
    RSVD_REQUIRE(n <= 64, "gemm_tn_skinny: n = %lld > 64", (long long)n);
    if (k == 0 || n == 0) return RSVD_OK;
    const int64_t S = tn_splits(m, k);
    RSVD_REQUIRE(ws_bytes >= S * k * n * (int64_t)sizeof(double), "gemm_tn_skinny: workspace too small");
    const int64_t rps = m > 0 ? cdiv(cdiv(m, S), kKc) * kKc : kKc;
    const int64_t splits = m > 0 ? cdiv(m, rps) : 1;  // m == 0: one split writes the zero partial
    dim3 grid((unsigned)splits, (unsigned)cdiv(k, 64));
    k_skinny_tn<<<grid, kSkThreads, 0, st>>>(m, (int)k, (int)n, A, lda, B, ldb, rps, (double*)ws, pred);
    RSVD_CHECK_LAUNCH();
    const int64_t tot = k * n;
    if (out_dtype == RSVD_F64)
        k_skinny_reduce<double><<<(unsigned)cdiv(tot, 32), 32 * kRedGroups, 0, st>>>(k, n, splits, (const double*)ws, alpha,
                                                                          beta, (double*)C, ldc, mu, cs, pred);
    else
        k_skinny_reduce<float><<<(unsigned)cdiv(tot, 32), 32 * kRedGroups, 0, st>>>(k, n, splits, (const double*)ws, alpha,
                                                                         beta, (float*)C, ldc, mu, cs, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace rsvd
