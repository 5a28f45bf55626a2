// tcgen05 3xTF32 tall-skinny GEMMs for the FP32 path (sm_100a).
//
//   NN:  C[m x n]  = alpha (A[m x k] B[k x n] - 1 row_sub^T) + beta C
//        operand A = A (K-major), K = k
//   TN:  C[k x n]  = alpha (A^T B - mu colsum^T) + beta C   (reduction over m)
//        operand A = A^T (MN-major: A's columns are contiguous), K = m, split
//        over K with FP64 reduction of the partials.
//   Operand B (the small d x p / n x p block) is split once by k_split_b into
//   two K-major planes [B_hi; B_lo] (row n = column n of B).
//
// FP32 accuracy from TF32 tensor cores by the hi/lo split
//   a = a_hi + a_lo, b = b_hi + b_lo  (hi = TF32 truncation, which the tensor
//   core applies to raw FP32 itself), a b ~= a_hi b_hi + a_hi b_lo + a_lo b_hi
//   as two MMAs per K=8 step: D0 | D1 += A_hi [B_hi | B_lo] (N = 2 BN) and
//   D0 += A_lo B_hi (N = BN); the drain sums D0 + D1.
// The TF32 tensor-core accumulator rounds with a bias (error measured to
// grow linearly in K: 4e-7 at K=32, 5e-6 at 1e3, 5e-5 at 1e4), so TMEM only
// accumulates KCHUNK = 4 k-blocks (K = 128); two accumulator sets alternate
// and four dedicated warps drain each finished chunk into round-to-nearest
// FP32 registers while the tensor core fills the other set.
// One kernel, k_tc_gemm_t, for every N tile: A_hi and A_lo live in TMEM (.ts
// MMAs). (An earlier BN 96 / 128 kernel with A_lo in shared memory was smem-
// bandwidth bound -- C4's A X 10.2 vs 8.3 ms -- and has been removed.)
#include <cuda.h>

#include <cmath>

#include "gemm.cuh"
#include "umma.cuh"

namespace rsvd {

namespace {

constexpr int BM = 128;      // UMMA M
constexpr int BK = 32;       // fp32 elements per 128-byte swizzle row
constexpr int KCHUNK = 4;  // k-blocks accumulated in TMEM before a drain

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4)                      // c_format F32
           | (2u << 7)                    // a_format TF32
           | (2u << 10)                   // b_format TF32
           | ((uint32_t)a_mn_major << 15) // a major
           | ((uint32_t)b_mn_major << 16) // b major
           | ((uint32_t)(N >> 3) << 17)   // N
           | ((uint32_t)(M >> 4) << 24);  // M
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// ------------------------------------------------------------------ kernels
struct TcParams {
    int64_t M, N, K;        // operand shapes: D[M x N] = Aop[M x K] Bop[K x N]
    int64_t k_per_split;    // K range per blockIdx.z (multiple of BK)
    int64_t Kp;             // padded K of the split-B planes (their row length)
    int64_t Np;             // rows per split-B plane (hi rows [0, Np), lo rows [Np, 2 Np))
    // epilogue
    int direct;             // 1: write C (NN); 0: FP32 partial to ws[z][M][N]
    float* C;
    int64_t ldc;
    double alpha, beta;
    const double* row_sub;
    float* ws;
    int64_t ldw;            // row pitch of the partials (multiple of 4 floats)
    int plain_vec;          // direct, alpha = 1, beta = 0, no row_sub, C rows 16-byte aligned
    int c_vec;              // direct and C rows 16-byte aligned (float4 epilogue with alpha/beta/row_sub)
    int sub_vec;            // direct, alpha = 1, beta = 0, row_sub, C rows 16-byte aligned, N % 4 == 0
    const int32_t* pred;
    int n_tiles;            // N tiles per M tile (blockIdx.x = m_tile * n_tiles + n_tile)
    // direct epilogue only: also write C's hi / lo planes in the k-blocked split-B
    // layout (k index = C's row), ready to be the B operand of a following TN
    // product -- instead of a k_split_b pass over C (read C, write 2 planes)
    float* emit;
    int64_t emit_np;        // rows per emitted plane (C's columns rounded up to 32)
};

// Profiling ablations (tools/ablate_tc.py builds variants; 0 in the product):
// 1 converters skip the split, 2 no MMAs issued, 4 drains skip the TMEM
// reads, 8 one MMA per k-step instead of two.
#ifndef RSVD_TC_ABLATE
#define RSVD_TC_ABLATE 0
#endif

// Pipeline trace (tools/trace_tc.py builds with -DRSVD_TC_TRACE): clock64
// stamps per k-block of CTA 0 and CTA kTraceCta2, 8 series each.
#ifdef RSVD_TC_TRACE
constexpr int kTraceKb = 512, kTraceCta2 = 200;
__device__ long long g_tc_trace[2][8][kTraceKb];
#define TC_TRACE(series, kb)                                                                      \
    do {                                                                                          \
        if ((blockIdx.x == 0 || blockIdx.x == kTraceCta2) && blockIdx.z == 0 && \
            (kb) < kTraceKb)                                                                       \
            g_tc_trace[blockIdx.x == 0 ? 0 : 1][series][kb] = clock64();                          \
    } while (0)
#else
#define TC_TRACE(series, kb) \
    do {                     \
    } while (0)
#endif

// Accumulator drain + epilogue. TMEM lane quarter
// q = warp % 4 holds tile rows 32q..32q+31; D0 | D1 (2 BN columns) of each
// finished chunk are summed into round-to-nearest FP32 registers.
template <int BN, bool MERGED = true>
__device__ __forceinline__ void drain_epilogue(const TcParams& p, uint32_t tmem_base, int warp, int lane, int nkb,
                                               int64_t m0, int64_t n0, uint64_t* acc_full, uint64_t* acc_empty) {
    const int quarter = warp % 4;
    const int64_t row = m0 + quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float sum[BN];
#pragma unroll
    for (int i = 0; i < BN; ++i) sum[i] = 0.f;
    const int nchunks = (nkb + KCHUNK - 1) / KCHUNK;
    for (int c = 0; c < nchunks; ++c) {
        const int set = c & 1;
        mbar_wait(&acc_full[set], (c >> 1) & 1);
        tc_fence_after();
        const uint32_t base = tmem_base + lane_off + set * (MERGED ? 2 : 1) * BN;
#pragma unroll
        for (int j = 0; j < ((RSVD_TC_ABLATE & 4) ? 0 : BN); j += 8) {
            float v0[8];
            tmem_ld8(base + j, v0);
            if constexpr (MERGED) {
                float v1[8];
                tmem_ld8(base + BN + j, v1);
#pragma unroll
                for (int i = 0; i < 8; ++i) sum[j + i] += v0[i] + v1[i];
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) sum[j + i] += v0[i];
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[set]);
    }
    if (warp % 4 == 3 && lane == 0) TC_TRACE(2, 511);
    // 16-byte stores where the layout allows: partials (padded pitch) and the
    // plain direct case; each lane owns one output row
    if (row < p.M && p.direct && p.sub_vec) {
        // centered A X (alpha = 1, beta = 0, row_sub): a compact float4 loop. The
        // general path below unrolls per-element branches over BN columns (~10k
        // SASS instructions at BN = 128): at C5 the instruction-cache misses of
        // that cold epilogue cost 40 % of the product (2.19 -> 3.10 ms).
        float* out = p.C + row * p.ldc + n0;
        const double* rs = p.row_sub + n0;
        const int ncols = (int)min((int64_t)BN, p.N - n0);
#pragma unroll
        for (int i = 0; i < BN; i += 4) {
            if (i < ncols) {
                const float4 v = make_float4((float)((double)sum[i] - rs[i]), (float)((double)sum[i + 1] - rs[i + 1]),
                                             (float)((double)sum[i + 2] - rs[i + 2]),
                                             (float)((double)sum[i + 3] - rs[i + 3]));
                *reinterpret_cast<float4*>(out + i) = v;
                sum[i] = v.x; sum[i + 1] = v.y; sum[i + 2] = v.z; sum[i + 3] = v.w;
            }
        }
    } else if (row < p.M && (!p.direct || p.plain_vec)) {
        float* out = p.direct ? p.C + row * p.ldc + n0 : p.ws + ((int64_t)blockIdx.z * p.M + row) * p.ldw + n0;
        const int ncols = (int)min((int64_t)BN, p.N - n0);
#pragma unroll
        for (int i = 0; i < BN; i += 4) {
            if (i + 4 <= ncols) {
                *reinterpret_cast<float4*>(out + i) = make_float4(sum[i], sum[i + 1], sum[i + 2], sum[i + 3]);
            } else {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (i + t < ncols) out[i + t] = sum[i + t];
            }
        }
    } else if (row < p.M) {
        // general direct epilogue; 16-byte loads/stores of 4 columns where the
        // layout allows (one lane per row: scalar accesses touched a separate
        // sector per element -- X -= Q C at n = 5e4: 47 us for a 40 MB product)
        const int ncols = (int)min((int64_t)BN, p.N - n0);
#pragma unroll
        for (int i = 0; i < BN; i += 4) {
            float* crow = p.C + row * p.ldc + n0 + i;
            if (p.direct && p.c_vec && i + 4 <= ncols) {
                float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
                if (p.beta != 0.0) cv = *reinterpret_cast<const float4*>(crow);
                const float cin[4] = {cv.x, cv.y, cv.z, cv.w};
                float res[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    double r = (double)sum[i + t];
                    if (p.row_sub) r -= p.row_sub[n0 + i + t];
                    r *= p.alpha;
                    if (p.beta != 0.0) r += p.beta * (double)cin[t];
                    res[t] = (float)r;
                }
                *reinterpret_cast<float4*>(crow) = make_float4(res[0], res[1], res[2], res[3]);
#pragma unroll
                for (int t = 0; t < 4; ++t) sum[i + t] = res[t];
            } else if (p.direct) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int64_t col = n0 + i + t;
                    if (i + t < ncols) {
                        double r = (double)sum[i + t];
                        if (p.row_sub) r -= p.row_sub[col];
                        r *= p.alpha;
                        if (p.beta != 0.0) r += p.beta * (double)p.C[row * p.ldc + col];
                        p.C[row * p.ldc + col] = (float)r;
                        sum[i + t] = (float)r;
                    }
                }
            }
        }
    }
    // sum[] now holds the stored values of this lane's row. Emission: lanes of a
    // warp are 32 consecutive rows of one 32-row k-block, so for a fixed column
    // the warp writes one contiguous 128-byte run per plane (rows past M, up to
    // the end of the last k-block, are written as zeros like k_split_b does)
    if (p.direct && p.emit != nullptr && row < (p.M + 31) / 32 * 32) {
        const int ncols = (int)min((int64_t)BN, p.N - n0);
        float* blk = p.emit + (row / 32) * (2 * p.emit_np) * 32 + (row % 32);
        const bool live = row < p.M;
#pragma unroll
        for (int i = 0; i < BN; ++i) {
            if (i < ncols) {
                const float x = live ? sum[i] : 0.f;
                const float h = tf32_hi(x);
                blk[(n0 + i) * 32] = h;
                blk[(p.emit_np + n0 + i) * 32] = tf32_rna(x - h);
            }
        }
    }
}

// ---- the kernel: both A halves in TMEM -------------------------------------
// Rings: A (smem, TMA, one 128 x 32 box per stage; freed by the converters as
// soon as they have read it), B (smem, TMA, [B_hi | B_lo] K-major for
// KPS = 2 k-blocks per slot; freed by the MMA commit) and T (TMEM columns
// [A_hi 64 | A_lo 64] for KPS k-blocks; written by the converters, freed by
// the MMA commit). An A smem stage is held only for the TMA latency plus one
// conversion, not for the tensor-core queue. Per K=8 step two .ts MMAs:
//   D0 | D1 += A_hi [B_hi | B_lo]   (N = 2 BN)
//   D0      += A_lo  B_hi           (N = BN)
// These MMAs are short (32-64 tensor cycles) and the tensor pipe queue is
// shallow, so the issuing thread must not stall: it runs alone (no warp
// divergence per step), waits on ONE barrier per slot of 2 k-blocks (the
// converters fold the B-arrival wait into t_full) and commits once per slot.
// Measured (tools/mma_rate_probe.cu): this stream is tensor-bound at 458
// cycles per k-block alone; a satisfied wait + fence per k-block adds ~110,
// busy neighbour warps ~175.
// Warps: 0 A producer, 1 MMA issuer (+TMEM alloc), 2 B producer, 3..6
// converters, 7..10 drain; warp % 4 gives each converter / drain warp its
// TMEM lane quarter.
constexpr int kTWarpDrain0 = 7, kTThreads = 32 * 11;
constexpr int KPS = 2;  // k-blocks per T / B slot

template <int BN, bool A_MN>
struct TmCfg {
    // BN <= 64: D0 | D1 += A_hi [B_hi | B_lo] merged into one N = 2 BN MMA.
    // BN >= 96: 2 x 2 BN accumulator columns would leave no TMEM for A, so
    // three N = BN MMAs accumulate into D0 alone (same tensor-pipe time).
    static constexpr bool MERGE = BN <= 64;
    static constexpr int A_BYTES = BM * BK * 4;        // 16 KB
    static constexpr int B_BYTES = BN * BK * 4;        // one plane's tile, one k-block
    static constexpr int B_SLOT = 2 * KPS * B_BYTES;    // [hi | lo] x KPS k-blocks
    static constexpr int ACC_COLS = (MERGE ? 4 : 2) * BN;  // 2 sets x (D0 | D1) or 2 sets x D0
    static constexpr int T_COLS = 2 * KPS * BK;         // [A_hi | A_lo] per slot
    static constexpr int T_STAGES = (512 - ACC_COLS) / T_COLS;
    static constexpr int B_STAGES = BN >= 112 ? 2 : (BN >= 64 ? 3 : 4);
    static constexpr int SMEM_BUDGET = (BN >= 96 ? 216 : 200) * 1024;  // 224 KB measured no faster
    static constexpr int A_STAGES_RAW = (SMEM_BUDGET - B_STAGES * B_SLOT) / A_BYTES;
    static constexpr int A_STAGES = A_STAGES_RAW > 12 ? 12 : A_STAGES_RAW;
    static constexpr int SMEM = A_STAGES * A_BYTES + B_STAGES * B_SLOT + 1024 + 512;
    static_assert(T_STAGES >= 2 && A_STAGES >= 2 * KPS, "pipeline too shallow");
    static_assert(KCHUNK % KPS == 0, "accumulator chunks must hold whole slots");
};

template <int BN, bool A_MN>
__global__ void __launch_bounds__(kTThreads, 1)
k_tc_gemm_t(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
    if (pred_off(p.pred)) return;
    if (threadIdx.x == 0) TC_TRACE(0, 511);
    using Cfg = TmCfg<BN, A_MN>;
    constexpr int SA = Cfg::A_STAGES, SB = Cfg::B_STAGES, ST = Cfg::T_STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a_ring = smem;
    uint8_t* b_ring = smem + SA * Cfg::A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(b_ring + SB * Cfg::B_SLOT);
    uint64_t* a_full = bars;
    uint64_t* a_empty = a_full + SA;
    uint64_t* b_full = a_empty + SA;
    uint64_t* b_empty = b_full + SB;
    uint64_t* t_full = b_empty + SB;
    uint64_t* t_empty = t_full + ST;
    uint64_t* acc_full = t_empty + ST;   // [2]
    uint64_t* acc_empty = acc_full + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // linear tile index, N tiles of one M tile adjacent (co-resident CTAs
    // share the A tile through L2 instead of streaming A once per N tile)
    const int64_t m0 = (int64_t)(blockIdx.x / p.n_tiles) * BM;
    const int64_t n0 = (int64_t)(blockIdx.x % p.n_tiles) * BN;
    const int64_t kbeg = (int64_t)blockIdx.z * p.k_per_split;
    const int64_t kend = min(p.K, kbeg + p.k_per_split);
    const int nkb = (int)((kend - kbeg + BK - 1) / BK);
    const int nslots = (nkb + KPS - 1) / KPS;  // the last slot may hold one k-block (zero-filled)

    if (threadIdx.x == 0) {
        for (int s = 0; s < SA; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 4);
        }
        for (int s = 0; s < SB; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int s = 0; s < ST; ++s) {
            mbar_init(&t_full[s], 4);
            mbar_init(&t_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) TC_TRACE(1, 511);
    const uint32_t t_col0 = tmem_base + Cfg::ACC_COLS;  // slot s: [hi 64 | lo 64] at t_col0 + T_COLS s

    if (warp == 0) {
        if (lane == 0) {  // ---------------- A producer (one k-block per stage; TMA zero-fills past K)
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < nslots * KPS; ++kb) {
                mbar_wait(&a_empty[s], ph ^ 1);
                TC_TRACE(0, kb);
                const int kk = (int)(kbeg + (int64_t)kb * BK);
                uint8_t* dst = a_ring + s * Cfg::A_BYTES;
                if (kb >= nkb) {
                    mbar_arrive(&a_full[s]);  // padding k-block of the last slot: converters write zeros
                } else if (mbar_expect_tx(&a_full[s], Cfg::A_BYTES), !A_MN) {
                    tma_load_2d(&tmA, &a_full[s], dst, kk, (int)m0);
                } else {
#pragma unroll
                    for (int i = 0; i < BM / 32; ++i)
                        tma_load_2d(&tmA, &a_full[s], dst + i * 32 * BK * 4, (int)(m0 + 32 * i), kk);
                }
                if (++s == SA) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {  // ---------------- B producer
            int s = 0;
            uint32_t ph = 0;
            for (int sl = 0; sl < nslots; ++sl) {
                mbar_wait(&b_empty[s], ph ^ 1);
                uint8_t* dst = b_ring + s * Cfg::B_SLOT;
                mbar_expect_tx(&b_full[s], Cfg::B_SLOT);
#pragma unroll
                for (int j = 0; j < KPS; ++j) {
                    const int kk = (int)(kbeg + (int64_t)(sl * KPS + j) * BK);
                    tma_load_3d(&tmB, &b_full[s], dst + j * 2 * Cfg::B_BYTES, 0, (int)n0, kk / BK);
                    tma_load_3d(&tmB, &b_full[s], dst + j * 2 * Cfg::B_BYTES + Cfg::B_BYTES, 0, (int)(p.Np + n0),
                                kk / BK);
                }
                if (++s == SB) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer (one thread, see above)
            constexpr uint32_t idesc2 = make_idesc(BM, 2 * BN, 0, 0);
            constexpr uint32_t idesc1 = make_idesc(BM, BN, 0, 0);
            const uint64_t db0 = make_desc(smem_u32(b_ring), 16, 1024, kLayoutSW128);
            constexpr uint64_t kSlotDesc = Cfg::B_SLOT >> 4;         // descriptor step per B slot
            constexpr uint64_t kKbDesc = (2 * Cfg::B_BYTES) >> 4;     // ... per k-block inside it
            int sb = 0, st = 0;
            uint32_t phb = 0, pht = 0;
            int chunk = 0;
            for (int sl = 0; sl < nslots; ++sl) {
                const int set = chunk & 1;
                const uint32_t d0 = tmem_base + set * (Cfg::MERGE ? 2 : 1) * BN;
                const bool first = (sl * KPS) % KCHUNK == 0;
                if (first) mbar_wait(&acc_empty[set], ((chunk >> 1) & 1) ^ 1);
                TC_TRACE(4, sl);
                mbar_wait(&t_full[st], pht);
                TC_TRACE(6, sl);
                tc_fence_after();
                const uint64_t db = db0 + sb * kSlotDesc;
                const uint32_t ta = t_col0 + st * Cfg::T_COLS;
#pragma unroll
                for (int j = 0; j < KPS; ++j) {
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        if (RSVD_TC_ABLATE & 2) continue;
                        const uint64_t dbk = db + j * kKbDesc + 2 * ks;
                        const uint32_t tk = ta + j * BK + ks * 8;
                        const uint32_t acc0 = (first && j == 0 && ks == 0) ? 0u : 1u;
                        if constexpr (Cfg::MERGE) {
                            tc_mma_tf32_ts(d0, tk, dbk, idesc2, acc0);  // D0 | D1 += A_hi [B_hi | B_lo]
                        } else {
                            tc_mma_tf32_ts(d0, tk, dbk, idesc1, acc0);                           // A_hi B_hi
                            tc_mma_tf32_ts(d0, tk, dbk + (Cfg::B_BYTES >> 4), idesc1, 1u);      // A_hi B_lo
                        }
                        if (RSVD_TC_ABLATE & 8) continue;
                        tc_mma_tf32_ts(d0, tk + KPS * BK, dbk, idesc1, 1u);  // D0 += A_lo B_hi
                    }
                }
                tc_commit(&t_empty[st]);
                tc_commit(&b_empty[sb]);
                if ((sl * KPS + KPS) % KCHUNK == 0 || sl == nslots - 1) {
                    tc_commit(&acc_full[set]);
                    ++chunk;
                }
                TC_TRACE(7, sl);
                if (++sb == SB) { sb = 0; phb ^= 1; }
                if (++st == ST) { st = 0; pht ^= 1; }
            }
        }
    } else if (warp < kTWarpDrain0) {
        // ---------------- converters: thread (quarter q, lane l) owns tile row
        // m = 32q + l = its TMEM lane; per slot it reads the row's 2 x 32 k
        // values from two A stages (freeing each at once), writes hi = raw A
        // (the tensor core truncates it to TF32) and lo = A - trunc_tf32(A)
        // (exact in FP32; truncated to TF32 by the tensor core, an error of
        // the order of the dropped a_lo b_lo term), then, once the slot's B
        // tiles have landed, hands the slot to the MMA thread.
        const int quarter = warp % 4;
        const int m = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        int sa = 0, sb = 0, st = 0;
        uint32_t pha = 0, phb = 0, pht = 0;
        for (int sl = 0; sl < nslots; ++sl) {
            mbar_wait(&t_empty[st], pht ^ 1);
            tc_fence_after();
            const uint32_t t = t_col0 + lane_off + st * Cfg::T_COLS;
#pragma unroll
            for (int j = 0; j < KPS; ++j) {
                mbar_wait(&a_full[sa], pha);
                if (warp == 4 && lane == 0) TC_TRACE(1, sl * KPS + j);
                const uint8_t* a = a_ring + sa * Cfg::A_BYTES;
                float x[32];
                if (sl * KPS + j >= nkb) {
#pragma unroll
                    for (int k = 0; k < 32; ++k) x[k] = 0.f;
                } else if (!A_MN) {
                    // K-major SWIZZLE_128B: row m = 128 bytes, 16B chunk c at c ^ (m % 8)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 v = *reinterpret_cast<const float4*>(a + m * 128 + ((c ^ (m & 7)) << 4));
                        x[4 * c + 0] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
                    }
                } else {
                    // MN-major SWIZZLE_128B_BASE32B: atom q (32 M x 32 K) at q*4096,
                    // K row k = 128 bytes, 32B chunk (l/8) at (l/8) ^ (k % 4)
                    const uint8_t* atom = a + quarter * 4096 + (lane & 7) * 4;
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        x[k] = *reinterpret_cast<const float*>(atom + k * 128 + (((lane >> 3) ^ (k & 3)) << 5));
                }
                // the stage is re-filled by TMA (async proxy) once released: the
                // generic reads above must be complete first. Without the proxy
                // fence ptxas issued the arrive ahead of the loads' completion
                // (per-row corruption when a refill landed early).
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_empty[sa]);
                float lo[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) lo[k] = (RSVD_TC_ABLATE & 1) ? 0.f : x[k] - tf32_hi(x[k]);
                tmem_st16(t + j * BK, x);
                tmem_st16(t + j * BK + 16, x + 16);
                tmem_st16(t + KPS * BK + j * BK, lo);
                tmem_st16(t + KPS * BK + j * BK + 16, lo + 16);
                if (++sa == SA) { sa = 0; pha ^= 1; }
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            mbar_wait(&b_full[sb], phb);
            __syncwarp();
            if (lane == 0) mbar_arrive(&t_full[st]);
            if (warp == 4 && lane == 0) TC_TRACE(3, sl);
            if (++sb == SB) { sb = 0; phb ^= 1; }
            if (++st == ST) { st = 0; pht ^= 1; }
        }
    } else {
        drain_epilogue<BN, Cfg::MERGE>(p, tmem_base, warp, lane, (nslots * KPS), m0, n0, acc_full, acc_empty);
        if (warp == kTWarpDrain0 && lane == 0) TC_TRACE(3, 511);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
}

// Split the operand B (K x N, ld) into two K-major planes, hi then lo, each
// Np x Kp (row n holds column n of B), zero padded so boxes past K or N read
// zeros, stored k-blocked: for k-block kb, rows [0, Np) of hi then [Np, 2 Np)
// of lo, 32 floats (128 bytes) each -> element (n, k) of plane P at
// ((kb * 2 Np) + P Np + n) * 32 + k % 32. One TMA box (32 k x BN rows) is
// then one contiguous 128 BN-byte run (a TN product streams B from HBM; the
// row-major plane made every box 128-byte pieces 4 Kp bytes apart).
// Transposes through a 32 x 33 shared tile.
// Grid-stride over the 32 x 32 tiles (at most a few CTAs per SM), so a
// launch whose device predicate is off retires in microseconds even when B
// is an n x p block (C4: 218k tiles). The next tile's loads are issued before
// the current tile is transposed and stored (register double buffer). Plane
// columns >= N are left unwritten: they only feed output columns >= n, which
// are never stored.
__global__ void __launch_bounds__(256) k_split_b(int64_t K, int64_t N, const float* __restrict__ B, int64_t ldb,
                                                 int64_t Kp, int64_t Np, float* __restrict__ out,
                                                 const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    __shared__ float t[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    const int64_t tk = Kp / 32, tiles = tk * (Np / 32);
    auto load = [&](int64_t tile, float (&v)[4]) {
        const int64_t k0 = (tile % tk) * 32, c0 = (tile / tk) * 32;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t r = k0 + ty + 8 * q, c = c0 + tx;
            v[q] = (r < K && c < N) ? __ldg(B + r * ldb + c) : 0.f;
        }
    };
    float cur[4], nxt[4];
    int64_t tile = blockIdx.x;
    if (tile < tiles) load(tile, cur);
    for (; tile < tiles; tile += gridDim.x) {
        const int64_t nt = tile + gridDim.x;
        if (nt < tiles) load(nt, nxt);
        const int64_t k0 = (tile % tk) * 32, c0 = (tile / tk) * 32;
#pragma unroll
        for (int q = 0; q < 4; ++q) t[ty + 8 * q][tx] = cur[q];
        __syncthreads();
        float* blk = out + (k0 / 32) * (2 * Np) * 32;  // k0 is a multiple of 32
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t c = c0 + ty + 8 * q;
            if (c < N) {
                const float x = t[tx][ty + 8 * q];
                const float h = tf32_hi(x);
                blk[c * 32 + tx] = h;
                blk[(Np + c) * 32 + tx] = tf32_rna(x - h);
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
    }
}

template <typename TO>
__global__ void k_tc_reduce(int64_t M, int64_t N, int64_t ldw, int64_t splits, const float* __restrict__ ws, double alpha,
                            double beta, TO* __restrict__ C, int64_t ldc, const double* __restrict__ mu,
                            const double* __restrict__ cs, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    int64_t r = e / N, c = e % N;
    double v = 0.0;
    for (int64_t s = 0; s < splits; ++s) v += (double)ws[(s * M + r) * ldw + c];
    if (mu) v -= mu[r] * cs[c];
    v *= alpha;
    if (beta != 0.0) v += beta * (double)C[r * ldc + c];
    C[r * ldc + c] = (TO)v;
}

// Same sum for outputs with few CTAs' worth of threads (projection-sized M):
// block = 32 outputs x 8 split groups, group g sums splits g, g + 8, ... and
// the group sums are added in group order (deterministic), so each thread
// issues splits / 8 loads instead of all of them back to back.
template <typename TO>
__global__ void __launch_bounds__(256)
k_tc_reduce_g(int64_t M, int64_t N, int64_t ldw, int64_t splits, const float* __restrict__ ws, double alpha,
              double beta, TO* __restrict__ C, int64_t ldc, const double* __restrict__ mu,
              const double* __restrict__ cs, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    __shared__ double part[8][33];
    const int o = threadIdx.x % 32, g = threadIdx.x / 32;
    const int64_t e = (int64_t)blockIdx.x * 32 + o;
    const bool ok = e < M * N;
    const int64_t r = ok ? e / N : 0, c = ok ? e % N : 0;
    double v = 0.0;
    if (ok)
        for (int64_t s = g; s < splits; s += 8) v += (double)ws[(s * M + r) * ldw + c];
    part[g][o] = v;
    __syncthreads();
    if (g != 0 || !ok) return;
    double t = part[0][o];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += part[i][o];
    if (mu) t -= mu[r] * cs[c];
    t *= alpha;
    if (beta != 0.0) t += beta * (double)C[r * ldc + c];
    C[r * ldc + c] = (TO)t;
}

// ------------------------------------------------------------------ host
// 2-D fp32 tensor map: inner dim (contiguous) x outer dim, box 32 x box_outer.
// mn_major selects the 32-byte-atom 128B swizzle the MN-major UMMA layout needs.
int make_map(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int64_t ld_elems, int box_outer,
             bool mn_major) {
    EncodeTiledFn fn = encode_fn();
    RSVD_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 4)};
    cuuint32_t box[2] = {32, (cuuint32_t)box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RSVD_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return RSVD_OK;
}

// k-blocked split-B planes (see k_split_b): dims {32, 2 Np, Kp / 32}, box
// {32, BN, 1}, 128B swizzle (the smem tile is the same K-major layout as a
// 2-D box of a row-major plane).
int make_map_b(CUtensorMap* map, const void* base, int64_t Kp, int64_t Np, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    RSVD_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {32, (cuuint64_t)(2 * Np), (cuuint64_t)(Kp / 32)};
    cuuint64_t strides[2] = {128, (cuuint64_t)(2 * Np * 128)};
    cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RSVD_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (split B) failed (%d)", (int)r);
    return RSVD_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int pick_bn(int64_t n) {
    // the kernel is instantiated for these widths (UMMA N: multiples of 16 at M = 128)
    if (n <= 32) return 32;
    if (n <= 64) return 64;
    if (n <= 96) return 96;
    // several N tiles: the width that pads the fewest MMA columns (n = 200: 2 x 112 = 224
    // instead of 2 x 128 = 256, 12.5 % fewer tensor-pipe cycles), wider on ties
    static const bool bn112 = !(getenv("RSVD_TC_BN112") && atoi(getenv("RSVD_TC_BN112")) == 0);
    int best = 128;
    int64_t best_cols = cdiv(n, 128) * 128;
    if (bn112 && cdiv(n, 112) * 112 < best_cols && cdiv(n, 112) == cdiv(n, 128)) best = 112;
    return best;
}

template <int BN, bool A_MN>
int launch_tc(const CUtensorMap& tA, const CUtensorMap& tB, const TcParams& p, dim3 grid, cudaStream_t st) {
    static PerDevice<bool> attr_dev;  // cudaFuncSetAttribute is per device
    bool& attr_set = attr_dev.get();
    using Cfg = TmCfg<BN, A_MN>;
    if (!attr_set) {
        RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_tc_gemm_t<BN, A_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Cfg::SMEM));
        attr_set = true;
    }
    k_tc_gemm_t<BN, A_MN><<<grid, kTThreads, Cfg::SMEM, st>>>(tA, tB, p);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

template <bool A_MN>
int dispatch_bn(int bn, const CUtensorMap& tA, const CUtensorMap& tB, const TcParams& p, dim3 grid,
                cudaStream_t st) {
    switch (bn) {
        case 32: return launch_tc<32, A_MN>(tA, tB, p, grid, st);
        case 64: return launch_tc<64, A_MN>(tA, tB, p, grid, st);
        case 96: return launch_tc<96, A_MN>(tA, tB, p, grid, st);
        case 112: return launch_tc<112, A_MN>(tA, tB, p, grid, st);
        default: return launch_tc<128, A_MN>(tA, tB, p, grid, st);
    }
}

// scratch for the split B array (grows; stream-ordered reuse)
struct Scratch {
    void* ptr = nullptr;
    size_t bytes = 0;
};

// Grow-only scratch. A superseded buffer is never freed: a CUDA graph captured
// earlier (GraphedFactorization, the public API's graph cache) holds its
// address, and a later, larger product must not free it under the graph.
float* scratch_get(Scratch& sc, size_t need, cudaStream_t st) {
    if (sc.bytes < need) {
        // geometric growth bounds the number of retired buffers (log1.5 of
        // the largest request) while keeping each one alive for old graphs
        const size_t grow = sc.bytes + sc.bytes / 2;
        if (need < grow) need = grow;
        void* p = nullptr;
        if (cudaMallocAsync(&p, need, st) != cudaSuccess) return nullptr;
        sc.ptr = p;  // the previous buffer stays allocated (see above)
        sc.bytes = need;
    }
    return (float*)sc.ptr;
}

int split_b(const float* B, int64_t K, int64_t N, int64_t ldb, int64_t Kp, int64_t Np, float* out,
            const int32_t* pred, cudaStream_t st) {
    const int64_t tiles = (Kp / 32) * (Np / 32);
    const int64_t cap = (int64_t)sm_count() * 8;
    k_split_b<<<(unsigned)(tiles < cap ? tiles : cap), dim3(32, 8), 0, st>>>(K, N, B, ldb, Kp, Np, out, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int64_t tn_splits_tc(int64_t Mop, int64_t Nop, int64_t Kop) {
    // split-K for parallelism (accuracy is handled by the chunked TMEM
    // accumulation), one CTA per (tile, split), at most one CTA per SM: the
    // smallest split count whose CTAs fill the SMs in waves >= 95% full (C2
    // A^T.Y: 79 tiles x 9 splits = 4.8 waves, vs 4 splits = 2.14 waves),
    // keeping >= 8 k-blocks per split and <= 64 partials
    if (const char* f = getenv("RSVD_TC_SPLITS")) return atoi(f) > 0 ? atoi(f) : 1;  // debugging override
    const int bn = pick_bn(Nop);
    const int64_t tiles = cdiv(Mop, BM) * cdiv(Nop, bn);
    const int64_t G = sm_count();
    const int64_t max_s = cdiv(Kop, 8 * BK) < 64 ? cdiv(Kop, 8 * BK) : 64;
    int64_t best = 1;
    double best_e = 0.0;
    for (int64_t S = 1; S <= max_s; ++S) {
        const double u = (double)(tiles * S) / (double)G;
        const double e = u / std::ceil(u);
        if (e > best_e + 1e-9) {
            best_e = e;
            best = S;
        }
        if (e >= 0.95) return S;
    }
    return best;
}


}  // namespace

bool gemm_tc_nn_supported(int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc, const void* A,
                          const void* B) {
    (void)ldb; (void)ldc; (void)B;
    if (getenv("RSVD_DISABLE_TC")) return false;
    return m >= BM && k >= BK && n >= 1 && (lda % 4) == 0 && aligned16(A) && m < (1ll << 31) && k < (1ll << 31);
}

int64_t split_planes_bytes(int64_t K, int64_t N) { return 2 * (cdiv(K, BK) * BK) * (cdiv(N, 32) * 32) * 4; }

int split_planes(int64_t K, int64_t N, const float* B, int64_t ldb, float* planes, const int32_t* pred,
                 cudaStream_t st) {
    if (K == 0 || N == 0) return RSVD_OK;
    return split_b(B, K, N, ldb, cdiv(K, BK) * BK, cdiv(N, 32) * 32, planes, pred, st);
}

int gemm_nn_tc(int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda, const float* B,
               int64_t ldb, double beta, float* C, int64_t ldc, const double* row_sub, const int32_t* pred,
               cudaStream_t st, float* emit) {
    int bn = pick_bn(n);
    // planes padded to 32 rows only: a last N tile's hi box may run into the lo
    // plane (and its lo box past 2 Np, zero-filled) -- those rows feed output
    // columns >= n, which are never stored
    const int64_t Kp = cdiv(k, BK) * BK, Np = cdiv(n, 32) * 32;
    static thread_local PerDevice<Scratch> sc_dev;  // split-B buffer, per device
    float* bs = scratch_get(sc_dev.get(), (size_t)(2 * Kp * Np * 4), st);
    RSVD_REQUIRE(bs != nullptr, "gemm_nn_tc: scratch allocation failed");
    int rc = split_b(B, k, n, ldb, Kp, Np, bs, pred, st);
    if (rc) return rc;
    CUtensorMap tA, tB;
    rc = make_map(&tA, A, k, m, lda, BM, false);
    if (rc) return rc;
    rc = make_map_b(&tB, bs, Kp, Np, bn);
    if (rc) return rc;
    TcParams p{};
    p.M = m; p.N = n; p.K = k; p.k_per_split = Kp; p.Kp = Kp; p.Np = Np;
    p.direct = 1; p.C = C; p.ldc = ldc; p.alpha = alpha; p.beta = beta; p.row_sub = row_sub; p.ws = nullptr;
    p.plain_vec = alpha == 1.0 && beta == 0.0 && row_sub == nullptr && ldc % 4 == 0 && aligned16(C);
    p.c_vec = ldc % 4 == 0 && aligned16(C);
    p.sub_vec = alpha == 1.0 && beta == 0.0 && row_sub != nullptr && ldc % 4 == 0 && n % 4 == 0 && aligned16(C);
    p.pred = pred;
    p.emit = emit;
    p.emit_np = cdiv(n, 32) * 32;
    p.n_tiles = (int)cdiv(n, bn);
    // (a split-K variant for wave balance -- C2: 391 tiles = 2.64 waves -- was
    // measured no faster: 2 / 3 / 4 splits 0.452 / 0.443 / 0.454 ms vs 0.441)
    dim3 grid((unsigned)(cdiv(m, BM) * p.n_tiles), 1, 1);
    return dispatch_bn<false>(bn, tA, tB, p, grid, st);
}

bool gemm_tc_tn_supported(int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, const void* A, const void* B) {
    (void)ldb; (void)B;
    if (getenv("RSVD_DISABLE_TC")) return false;
    // any output height: the A^T tile rows past k are TMA zero-fill
    return k >= 8 && m >= BK && n >= 1 && (lda % 4) == 0 && aligned16(A) && m < (1ll << 31) && k < (1ll << 31);
}

int64_t gemm_tn_tc_ws_bytes(int64_t m, int64_t n, int64_t k) {
    int64_t s = tn_splits_tc(k, n, m);
    return s * k * cdiv(n, 4) * 4 * 4 + 256;  // partial rows padded to 16 bytes
}

int gemm_tn_tc(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda,
               const float* B, int64_t ldb, double beta, void* C, int64_t ldc, const double* mu, const double* cs,
               void* ws, int64_t ws_bytes, const int32_t* pred, cudaStream_t st, const float* b_planes) {
    // operand view: D[Mop x Nop] = A^T[Mop x Kop] B[Kop x Nop], Mop = k, Kop = m
    const int64_t Mop = k, Nop = n, Kop = m;
    int bn = pick_bn(Nop);
    const int64_t S = tn_splits_tc(Mop, Nop, Kop);
    RSVD_REQUIRE(ws_bytes >= S * Mop * cdiv(Nop, 4) * 4 * 4, "gemm_tn_tc: workspace too small");
    RSVD_REQUIRE(aligned16(ws), "gemm_tn_tc: workspace must be 16-byte aligned");
    const int64_t Kp = cdiv(Kop, BK) * BK, Np = cdiv(Nop, 32) * 32;  // see gemm_nn_tc
    // B already split by the caller (planes emitted by the NN product that wrote B,
    // or rsvd_split_planes): no pass over B here
    const float* bs = b_planes;
    int rc = RSVD_OK;
    if (bs == nullptr) {
        static thread_local PerDevice<Scratch> sc_dev;
        float* sb = scratch_get(sc_dev.get(), (size_t)(2 * Kp * Np * 4), st);
        RSVD_REQUIRE(sb != nullptr, "gemm_tn_tc: scratch allocation failed");
        rc = split_b(B, Kop, Nop, ldb, Kp, Np, sb, pred, st);
        if (rc) return rc;
        bs = sb;
    }
    CUtensorMap tA, tB;
    rc = make_map(&tA, A, k /*inner = columns of A*/, m, lda, BK, true);
    if (rc) return rc;
    rc = make_map_b(&tB, bs, Kp, Np, bn);
    if (rc) return rc;
    TcParams p{};
    p.M = Mop; p.N = Nop; p.K = Kop; p.Np = Np;
    p.k_per_split = cdiv(cdiv(Kop, S), BK) * BK;
    p.Kp = Kp;
    p.direct = 0; p.ws = (float*)ws; p.pred = pred;
    p.ldw = cdiv(Nop, 4) * 4;
    p.n_tiles = (int)cdiv(Nop, bn);
    dim3 grid((unsigned)(cdiv(Mop, BM) * p.n_tiles), 1, (unsigned)S);
    rc = dispatch_bn<true>(bn, tA, tB, p, grid, st);
    if (rc) return rc;
    int64_t tot = Mop * Nop;
    // few outputs, many splits (projection coefficients): split-grouped reduce
    const bool grouped = S >= 16 && tot * 8 <= (int64_t)sm_count() * 2048;
    if (grouped) {
        if (out_dtype == RSVD_F64)
            k_tc_reduce_g<double><<<(unsigned)cdiv(tot, 32), 256, 0, st>>>(Mop, Nop, p.ldw, S, (const float*)ws, alpha,
                                                                            beta, (double*)C, ldc, mu, cs, pred);
        else
            k_tc_reduce_g<float><<<(unsigned)cdiv(tot, 32), 256, 0, st>>>(Mop, Nop, p.ldw, S, (const float*)ws, alpha,
                                                                           beta, (float*)C, ldc, mu, cs, pred);
    } else if (out_dtype == RSVD_F64)
        k_tc_reduce<double><<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(Mop, Nop, p.ldw, S, (const float*)ws, alpha, beta,
                                                                       (double*)C, ldc, mu, cs, pred);
    else
        k_tc_reduce<float><<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(Mop, Nop, p.ldw, S, (const float*)ws, alpha, beta,
                                                                      (float*)C, ldc, mu, cs, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace rsvd

#ifdef RSVD_TC_TRACE
extern "C" int rsvd_debug_tc_trace(long long* host_out) {
    return (int)cudaMemcpyFromSymbol(host_out, rsvd::g_tc_trace, sizeof(rsvd::g_tc_trace));
}
#endif
