// FP64 tensor-core (DMMA, `mma.sync.m16n8k4.f64`) tall-skinny products: the
// oracle-parity precision path (north_star subsystem 1).
// tcgen05 has no FP64 kind, so FP64 MMAs are warp-synchronous mma.sync fed
// from a 3-stage cp.async shared-memory ring.
//
//   gemm_nn:  C = alpha (A B - 1 row_sub^T) + beta C     A m x k, B k x n
//   gemm_tn:  C = alpha (A^T B - mu colsum^T) + beta C   reduction over m in
//             fixed row splits, FP64 partials reduced in split order
//             (deterministic, like the SIMT kernel it replaces).
//
// Replaces the FP64 `mm` of _kernels.pyx:56-71 as called through
// MatrixOperator.apply / apply_transpose (matrix.py:227-247), the projections
// of _mgs (factor.py:93-98) and post_process's products (rsvd.py:212-219).
//
// One kernel body serves both products: NN stages an A tile as
// [m rows][k cols] and reads fragments row-major; TN stages [reduction rows]
// [output cols] straight from A's rows and reads fragments transposed. Row
// strides are padded by 4 doubles so each half-warp's 8-byte fragment loads
// hit 16 distinct bank pairs.
#include "common.cuh"
#include "gemm.cuh"
#include <stdlib.h>

namespace rsvd {

namespace {

constexpr int kThreads = 256;  // 8 warps
constexpr int kStages = 3;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? 8 : 0;  // src-size 0 zero-fills the destination
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
// 16-byte copy of two doubles; src_bytes 16, 8 (second zero-filled) or 0.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double* c, double a0, double a1, double b0) {
    asm(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

// m16n8k16: A fragment a[2h + j] = A(g + 8 j, t + 4 h), B fragment
// b[h] = B(t + 4 h, g), h = 0..3 -- four k4 steps in one instruction.
__device__ __forceinline__ void dmma16(double* c, const double* a, const double* b) {
    asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
        "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
          "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

#ifndef RSVD_DMMA_K
#define RSVD_DMMA_K 16
#endif

// Tile config: BM output rows x BN output cols per CTA, BK reduction depth per
// stage; warps laid out WGM x WGN, each owning (BM/WGM) x (BN/WGN).
template <int BM, int BN, int BK, int WGM>
struct DmmaCfg {
    static constexpr int WGM_ = WGM, WGN = 8 / WGM;
    static constexpr int WTM = BM / WGM, WTN = BN / WGN;
    static constexpr int FM = WTM / 16, FN = WTN / 8;  // m16 / n8 fragments per warp
    static_assert(WGM * WGN == 8 && FM >= 1 && FN >= 1, "bad warp layout");
};

// TRANS = false: C tile = A[m0:m0+BM, kr] * B[kr, n0:n0+BN]   (NN, kr = k range)
// TRANS = true : C tile = A[kr, m0:m0+BM]^T * B[kr, n0:n0+BN] (TN, kr = a row split)
// For TN "m" below is the output row count (the caller's k) and "kred" the
// reduction length (the caller's m).
// VEC: operands 16-byte aligned with even leading dimensions -> 16-byte
// cp.async of column pairs (tile origins are even), else 8-byte copies.
template <bool TRANS, bool VEC, int BM, int BN, int BK, int WGM>
__global__ void __launch_bounds__(kThreads, 2)
k_dmma(int64_t mout, int64_t n, int64_t kred, const double* __restrict__ A, int64_t lda,
       const double* __restrict__ B, int64_t ldb, int64_t red_per_split, double alpha, double beta,
       double* __restrict__ C, int64_t ldc, const double* __restrict__ row_sub,
       double* __restrict__ ws, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    using Cfg = DmmaCfg<BM, BN, BK, WGM>;
    // A stage: NN [BM][BK + 4]; TN [BK][BM + 4]. B stage: [BK][BN + 4].
    constexpr int SA = TRANS ? BM + 4 : BK + 4;
    constexpr int A_ELEMS = TRANS ? BK * SA : BM * SA;
    constexpr int SB = BN + 4;
    constexpr int B_ELEMS = BK * SB;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + kStages * A_ELEMS;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp % Cfg::WGM_, wn = warp / Cfg::WGM_;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    const int64_t rbeg = (int64_t)blockIdx.z * red_per_split;
    const int64_t rend = min(kred, rbeg + red_per_split);
    const int64_t nsteps = rend > rbeg ? (rend - rbeg + BK - 1) / BK : 0;

    // n8 fragments entirely past n are computed (zero B) but not stored
    bool fn_live[Cfg::FN];
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) fn_live[j] = n0 + wn * Cfg::WTN + j * 8 < n;

    double acc[Cfg::FM][Cfg::FN][4];
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

    // stage a rows x cols block of M (row-major, ld) at (gr0, gc0) into dst
    // (row stride SD); rows >= rlim / cols >= clim are zero-filled
    auto stage = [&](double* dst, int SD, int rows, int cols, const double* M, int64_t ld, int64_t gr0,
                     int64_t gc0, int64_t rlim, int64_t clim) {
        if (VEC) {
            const int cp = cols / 2;
            for (int idx = threadIdx.x; idx < rows * cp; idx += kThreads) {
                int r = idx / cp, c = 2 * (idx % cp);
                int64_t gr = gr0 + r, gc = gc0 + c;
                int bytes = (gr < rlim && gc < clim) ? (gc + 1 < clim ? 16 : 8) : 0;
                cp_async16(dst + r * SD + c, bytes ? M + gr * ld + gc : M, bytes);
            }
        } else {
            for (int idx = threadIdx.x; idx < rows * cols; idx += kThreads) {
                int r = idx / cols, c = idx % cols;
                int64_t gr = gr0 + r, gc = gc0 + c;
                bool ok = gr < rlim && gc < clim;
                cp_async8(dst + r * SD + c, ok ? M + gr * ld + gc : M, ok);
            }
        }
    };
    auto load_stage = [&](int64_t step, int slot) {
        const int64_t r0 = rbeg + step * BK;
        double* as = As + slot * A_ELEMS;
        double* bs = Bs + slot * B_ELEMS;
        if (!TRANS)
            stage(as, SA, BM, BK, A, lda, m0, r0, mout, rend);
        else
            stage(as, SA, BK, BM, A, lda, r0, m0, rend, mout);
        stage(bs, SB, BK, BN, B, ldb, r0, n0, rend, n);
    };

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nsteps) load_stage(s, s);
        cp_async_commit();
    }
    for (int64_t step = 0; step < nsteps; ++step) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        // refill the slot consumed last iteration (all warps are past it)
        if (step + kStages - 1 < nsteps) load_stage(step + kStages - 1, (int)((step + kStages - 1) % kStages));
        cp_async_commit();
        const int slot = (int)(step % kStages);
        const double* as = As + slot * A_ELEMS;
        const double* bs = Bs + slot * B_ELEMS;
#if RSVD_DMMA_K == 16
        static_assert(BK % 16 == 0, "BK must be a multiple of 16");
#pragma unroll
        for (int kk = 0; kk < BK; kk += 16) {
            double af[Cfg::FM][8], bf[Cfg::FN][4];
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i) {
                const int r = wm * Cfg::WTM + i * 16 + g;
#pragma unroll
                for (int h = 0; h < 4; ++h)
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        af[i][2 * h + j] = TRANS ? as[(kk + t + 4 * h) * SA + r + 8 * j]
                                                 : as[(r + 8 * j) * SA + kk + t + 4 * h];
            }
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
                for (int h = 0; h < 4; ++h) bf[j][h] = bs[(kk + t + 4 * h) * SB + wn * Cfg::WTN + j * 8 + g];
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::FN; ++j) dmma16(acc[i][j], af[i], bf[j]);
        }
#else
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a0[Cfg::FM], a1[Cfg::FM], b0[Cfg::FN];
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i) {
                const int r = wm * Cfg::WTM + i * 16 + g;
                if (!TRANS) {
                    a0[i] = as[r * SA + kk + t];
                    a1[i] = as[(r + 8) * SA + kk + t];
                } else {
                    a0[i] = as[(kk + t) * SA + r];
                    a1[i] = as[(kk + t) * SA + r + 8];
                }
            }
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j) b0[j] = bs[(kk + t) * SB + wn * Cfg::WTN + j * 8 + g];
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j], a0[i], a1[i], b0[j]);
        }
#endif
    }
    cp_async_wait<0>();

    // epilogue: c0,c1 at (g, 2t..2t+1), c2,c3 at (g+8, 2t..2t+1)
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
            if (!fn_live[j]) continue;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t r = m0 + wm * Cfg::WTM + i * 16 + g + (v >= 2 ? 8 : 0);
                const int64_t c = n0 + wn * Cfg::WTN + j * 8 + 2 * t + (v & 1);
                if (r >= mout || c >= n) continue;
                double x = acc[i][j][v];
                if (TRANS) {
                    ws[((int64_t)blockIdx.z * mout + r) * n + c] = x;
                } else {
                    if (row_sub) x -= row_sub[c];
                    x *= alpha;
                    if (beta != 0.0) x += beta * C[r * ldc + c];
                    C[r * ldc + c] = x;
                }
            }
        }
}

template <typename TO>
__global__ void k_dmma_tn_reduce(int64_t k, int64_t n, int64_t splits, const double* __restrict__ ws,
                                 double alpha, double beta, TO* __restrict__ C, int64_t ldc,
                                 const double* __restrict__ mu, const double* __restrict__ cs,
                                 const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * n) return;
    int64_t r = idx / n, c = idx % n;
    double v = 0.0;
    for (int64_t s = 0; s < splits; ++s) v += ws[s * k * n + idx];  // fixed split order
    if (mu) v -= mu[r] * cs[c];
    v *= alpha;
    if (beta != 0.0) v += beta * (double)C[r * ldc + c];
    C[r * ldc + c] = (TO)v;
}

template <bool TRANS, int BM, int BN, int BK>
constexpr int dmma_smem() {
    return kStages * (((TRANS ? BK * (BM + 4) : BM * (BK + 4))) + BK * (BN + 4)) * (int)sizeof(double);
}

template <bool TRANS, bool VEC, int BM, int BN, int BK, int WGM>
int launch_one(dim3 grid, cudaStream_t st, int64_t mout, int64_t n, int64_t kred, const double* A,
               int64_t lda, const double* B, int64_t ldb, int64_t rps, double alpha, double beta, double* C,
               int64_t ldc, const double* row_sub, double* ws, const int32_t* pred) {
    constexpr int smem = dmma_smem<TRANS, BM, BN, BK>();
    auto kern = k_dmma<TRANS, VEC, BM, BN, BK, WGM>;
    static PerDevice<bool> attr_dev;  // per instantiation and device; idempotent
    bool& attr = attr_dev.get();
    if (!attr) {
        RSVD_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    kern<<<grid, kThreads, smem, st>>>(mout, n, kred, A, lda, B, ldb, rps, alpha, beta, C, ldc, row_sub,
                                       ws, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

template <bool TRANS, int BM, int BN, int BK, int WGM>
int launch(bool vec, dim3 grid, cudaStream_t st, int64_t mout, int64_t n, int64_t kred, const double* A,
           int64_t lda, const double* B, int64_t ldb, int64_t rps, double alpha, double beta, double* C,
           int64_t ldc, const double* row_sub, double* ws, const int32_t* pred) {
    if (vec)
        return launch_one<TRANS, true, BM, BN, BK, WGM>(grid, st, mout, n, kred, A, lda, B, ldb, rps, alpha,
                                                         beta, C, ldc, row_sub, ws, pred);
    return launch_one<TRANS, false, BM, BN, BK, WGM>(grid, st, mout, n, kred, A, lda, B, ldb, rps, alpha,
                                                      beta, C, ldc, row_sub, ws, pred);
}

bool vec_ok(const double* A, int64_t lda, const double* B, int64_t ldb) {
    return ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) && lda % 2 == 0 && ldb % 2 == 0;
}

constexpr int NN_BK = 16;
// TN: 128 output rows x 64 cols, 16 reduction rows per stage.
constexpr int TN_BM = 128, TN_BN = 64, TN_BK = 16;
constexpr int kCtasPerSm = 2;

// Row splits for A^T B: enough CTAs for >= 2 waves, the count chosen so the
// last wave is nearly full (wave quantisation dominates at C2: 79 tiles).
int64_t dmma_tn_splits(int64_t m, int64_t n, int64_t k) {
    const int64_t tiles = cdiv(k, TN_BM) * cdiv(n, TN_BN);
    const int64_t slots = (int64_t)sm_count() * kCtasPerSm;
    int64_t max_s = cdiv(m, 256);
    if (max_s < 1) max_s = 1;
    int64_t best = 1;
    double best_score = -1.0;
    for (int64_t s = 1; s <= max_s && s <= 64; ++s) {
        const int64_t ctas = tiles * s;
        const int64_t waves = cdiv(ctas, slots);
        const double eff = (double)ctas / (double)(waves * slots);
        // prefer full waves; past 4 waves more splits only add partial traffic
        const double score = eff * (waves >= 2 ? 1.0 : 0.75 + 0.25 * (double)ctas / slots) - 0.01 * (waves > 4);
        if (score > best_score + 1e-9) {
            best_score = score;
            best = s;
        }
    }
    return best;
}

// Small right factor (k, n <= 64): C = alpha (A B - 1 row_sub^T) + beta C with
// one thread per output row on the FP64 CUDA cores (B in shared memory, read
// as broadcasts; 32 accumulators per pass). An A/B variant only: slower than
// the DMMA tiles at 50000 x 50 x 50 (52 vs 31 us).
constexpr int kSmallRows = 128;

__global__ void __launch_bounds__(kSmallRows)
k_dnn_small(int64_t m, int n, int k, double alpha, const double* __restrict__ A, int64_t lda,
            const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
            const double* __restrict__ row_sub, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    __shared__ double Bs[64][64];
    for (int idx = threadIdx.x; idx < k * n; idx += blockDim.x) Bs[idx / n][idx % n] = B[(int64_t)(idx / n) * ldb + idx % n];
    __syncthreads();
    const int64_t row = (int64_t)blockIdx.x * kSmallRows + threadIdx.x;
    if (row >= m) return;
    const double* a = A + row * lda;
    double* c = C + row * ldc;
    for (int h = 0; h < n; h += 32) {
        double acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.0;
#pragma unroll 2
        for (int kk = 0; kk < k; ++kk) {
            const double av = __ldg(a + kk);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = fma(av, Bs[kk][(h + j) & 63], acc[j]);
        }
        double cin[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) cin[j] = (beta != 0.0 && h + j < n) ? c[h + j] : 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (h + j < n) {
                double x = acc[j];
                if (row_sub) x -= row_sub[h + j];
                x *= alpha;
                if (beta != 0.0) x += beta * cin[j];
                c[h + j] = x;
            }
        }
    }
}

}  // namespace

int gemm_nn_dmma(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                 const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                 const double* row_sub, const int32_t* pred, cudaStream_t st) {
    if (m == 0 || n == 0) return RSVD_OK;
    // (RSVD_DNN_SMALL=1: the CUDA-core variant; measured 52 us vs 31 us for the
    // DMMA tiles at 50000 x 50 x 50, kept for A/B)
    static const bool small = getenv("RSVD_DNN_SMALL") != nullptr;
    if (small && n <= 64 && k <= 64) {
        k_dnn_small<<<(unsigned)cdiv(m, kSmallRows), kSmallRows, 0, st>>>(m, (int)n, (int)k, alpha, A, lda, B, ldb,
                                                                           beta, C, ldc, row_sub, pred);
        RSVD_CHECK_LAUNCH();
        return RSVD_OK;
    }
    const bool vec = vec_ok(A, lda, B, ldb);
    const int64_t slots = (int64_t)sm_count() * kCtasPerSm;
    if (n <= 32) {
        // 128 x 32 tiles, warps 8 x 1 (16 x 32 each): narrow blocks (C1: p = 20)
        dim3 grid((unsigned)cdiv(m, 128), (unsigned)cdiv(n, 32), 1);
        return launch<false, 128, 32, NN_BK, 8>(vec, grid, st, m, n, k, A, lda, B, ldb, k, alpha, beta, C, ldc,
                                                row_sub, nullptr, pred);
    }
    const int64_t ntn = cdiv(n, 64);
    if (cdiv(m, 128) * ntn < 3 * slots) {
        // too few 128-row tiles for full waves (C2 chain: 391 on 296 slots):
        // 64 x 64 tiles, warps 2 x 4 (32 x 16 each)
        dim3 grid((unsigned)cdiv(m, 64), (unsigned)ntn, 1);
        return launch<false, 64, 64, NN_BK, 2>(vec, grid, st, m, n, k, A, lda, B, ldb, k, alpha, beta, C, ldc,
                                               row_sub, nullptr, pred);
    }
    // 128 x 64 tiles, warps 4 x 2 (32 x 32 each)
    dim3 grid((unsigned)cdiv(m, 128), (unsigned)ntn, 1);
    return launch<false, 128, 64, NN_BK, 4>(vec, grid, st, m, n, k, A, lda, B, ldb, k, alpha, beta, C, ldc,
                                            row_sub, nullptr, pred);
}

// Outputs of at most 64 x 64 (Grams and small projections of an n x p block):
// one 64 x 64 tile, the reduction spread over ~one wave of CTAs (>= 128 rows
// each). The general path capped the split count at 64 CTAs for a single tile
// (C2 Gram 50000 x 50: 97 us on 64 of 296 CTA slots).
bool dmma_tn_small(int64_t n, int64_t k) { return k <= 64 && n <= 64; }

int64_t dmma_tn_small_splits(int64_t m) {
    const int64_t slots = (int64_t)sm_count() * kCtasPerSm;
    int64_t s = cdiv(m, 128);
    if (s > slots) s = slots;
    if (s < 1) s = 1;
    const int64_t rps = cdiv(cdiv(m, s), TN_BK) * TN_BK;
    return cdiv(m, rps) < 1 ? 1 : cdiv(m, rps);
}

// Split-ordered sum of many partials (grouped: 32 outputs x 8 split groups
// per CTA, group sums added in group order -- deterministic).
template <typename TO>
__global__ void __launch_bounds__(256)
k_dmma_tn_reduce_g(int64_t k, int64_t n, int64_t splits, const double* __restrict__ ws, double alpha, double beta,
                   TO* __restrict__ C, int64_t ldc, const double* __restrict__ mu, const double* __restrict__ cs,
                   const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    __shared__ double part[8][33];
    const int o = threadIdx.x % 32, g = threadIdx.x / 32;
    const int64_t e = (int64_t)blockIdx.x * 32 + o;
    const bool ok = e < k * n;
    double v = 0.0;
    if (ok)
        for (int64_t s = g; s < splits; s += 8) v += ws[s * k * n + e];
    part[g][o] = v;
    __syncthreads();
    if (g != 0 || !ok) return;
    double t = part[0][o];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += part[i][o];
    const int64_t r = e / n, c = e % n;
    if (mu) t -= mu[r] * cs[c];
    t *= alpha;
    if (beta != 0.0) t += beta * (double)C[r * ldc + c];
    C[r * ldc + c] = (TO)t;
}

int64_t gemm_tn_dmma_ws_bytes(int64_t m, int64_t n, int64_t k) {
    const int64_t s = dmma_tn_small(n, k) ? dmma_tn_small_splits(m) : dmma_tn_splits(m, n, k);
    return s * k * n * (int64_t)sizeof(double);
}

int gemm_tn_dmma(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                 int64_t lda, const double* B, int64_t ldb, double beta, void* C, int64_t ldc,
                 const double* mu, const double* cs, void* ws, int64_t ws_bytes, const int32_t* pred,
                 cudaStream_t st) {
    if (k == 0 || n == 0) return RSVD_OK;
    if (dmma_tn_small(n, k)) {
        const int64_t s = dmma_tn_small_splits(m);
        RSVD_REQUIRE(ws_bytes >= s * k * n * (int64_t)sizeof(double), "gemm_tn(dmma): workspace too small");
        const int64_t rps = cdiv(cdiv(m, s), TN_BK) * TN_BK;
        dim3 grid(1, 1, (unsigned)s);
        int rc = launch<true, 64, 64, TN_BK, 2>(vec_ok(A, lda, B, ldb), grid, st, k, n, m, A, lda, B, ldb, rps, 1.0,
                                                0.0, nullptr, 0, nullptr, (double*)ws, pred);
        if (rc != RSVD_OK) return rc;
        const unsigned nb = (unsigned)cdiv(k * n, 32);
        if (out_dtype == RSVD_F64)
            k_dmma_tn_reduce_g<double><<<nb, 256, 0, st>>>(k, n, s, (const double*)ws, alpha, beta, (double*)C, ldc,
                                                           mu, cs, pred);
        else
            k_dmma_tn_reduce_g<float><<<nb, 256, 0, st>>>(k, n, s, (const double*)ws, alpha, beta, (float*)C, ldc,
                                                          mu, cs, pred);
        RSVD_CHECK_LAUNCH();
        return RSVD_OK;
    }
    int64_t s = dmma_tn_splits(m, n, k);
    RSVD_REQUIRE(ws_bytes >= s * k * n * (int64_t)sizeof(double), "gemm_tn(dmma): workspace too small");
    int64_t rps = cdiv(cdiv(m, s), TN_BK) * TN_BK;
    dim3 grid((unsigned)cdiv(k, TN_BM), (unsigned)cdiv(n, TN_BN), (unsigned)s);
    int rc = launch<true, TN_BM, TN_BN, TN_BK, 4>(vec_ok(A, lda, B, ldb), grid, st, k, n, m, A, lda, B, ldb, rps,
                                                   1.0, 0.0, nullptr, 0, nullptr, (double*)ws, pred);
    if (rc != RSVD_OK) return rc;
    int64_t tot = k * n;
    unsigned nb = (unsigned)cdiv(tot, 256);
    if (out_dtype == RSVD_F64)
        k_dmma_tn_reduce<double><<<nb, 256, 0, st>>>(k, n, s, (const double*)ws, alpha, beta, (double*)C, ldc,
                                                     mu, cs, pred);
    else
        k_dmma_tn_reduce<float><<<nb, 256, 0, st>>>(k, n, s, (const double*)ws, alpha, beta, (float*)C, ldc,
                                                    mu, cs, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace rsvd
