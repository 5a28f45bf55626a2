// FP64-accurate products of an FP32 A on the int8 tensor cores (sm_100a,
// tcgen05 kind::i8): the Ozaki splitting scheme with exact int32 accumulation.
//
// Why: the reference builds its block-Krylov basis from normalized power
// blocks whose newest directions sit ~1e-11 below the block norm
// (rsvd.py:244-260, factor.py:79-118). Reproducing its sigma to 1e-4 needs
// products accurate to ~1e-15 relative (measured on the C2 matrix: product
// noise 1e-15 -> sigma 1.7e-6 off, 1e-13 -> 1.4e-4 and different deflation
// decisions). 3xTF32 gives ~1e-7; FP64 DMMA gives 1e-16 at ~37 TFLOP/s.
//
// Scheme (per product D = A X, A FP32 n x d held in HBM as slices):
//   * every row r of A is scaled by 2^-E_r (2^E_r > ~2 max_c |A[r,c]|), rounded
//     to a 40-bit integer N = rint(A[r,c] 2^(40 - E_r)) and written as SA = 5
//     signed base-256 digits: N = sum_i a_i 256^(4-i), a_i in [-128, 127]
//     (the bytes of (N + B) ^ B with B = 0x8080808080: adding 128 at every
//     byte position turns balanced digits into plain bytes). Exact for every
//     entry >= 2^-15 of the row maximum (FP32 carries 24 bits), rounded at
//     2^-41 of the row scale below that;
//   * every column c of the FP64 operand X likewise into SB = 6 digits (48
//     bits) with its own exponent F_c;
//   * D = 2^(E_r + F_c - 16) sum_{i+j <= 5} 2^-8(i+j) (a_i x_j): 20 int8 GEMMs
//     whose int32 sums are EXACT (|digit products| <= 2^14, at most 7 pairs
//     per level, K <= 16384 per CTA keeps every level below 2^31); the levels
//     are combined in FP64 in the epilogue. Neglected terms are ~2^-49 of
//     (row scale x column scale) per entry: FP64-class accuracy.
//     (Round 2 first used base-128 digits in [-64, 64] -- 6 x 7 digits, 27
//     GEMMs; a round-to-nearest base-256 digit can be +128, which int8 cannot
//     hold. Rounding to an integer first and taking its signed base-256 digits
//     from the least significant end keeps every digit in [-128, 127]: 26 %
//     fewer MMAs and 17 % fewer plane bytes at the same dropped-term size.)
//   * A^T Y uses the same row-scaled slices: A^T Y = sum_r (2^-E_r A[r,:])^T
//     (2^E_r Y[r,:]); the row scale is folded into Y before it is sliced, so
//     the A operand is read in place as an MN-major int8 tile.
// Per K = 32 step one A digit plane i multiplies the stacked digit planes
// [x_0 | x_1 | ... | x_(5-i)] (N = (6-i) BN, split into <= 256-column MMAs)
// into TMEM columns [i BN, 6 BN): level L = i + j accumulates at column L BN
// without any per-pair bookkeeping. TMEM holds all 6 levels (384 columns at
// BN = 64) for the whole K range of the CTA; the epilogue reads them once.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gemm.cuh"
#include "umma.cuh"

namespace rsvd {

namespace {

constexpr int OZ_BM = 128;
constexpr int OZ_KS = 32;        // int8 K per MMA = bytes per smem tile row
constexpr int OZ_DB = 8;         // bits per digit (signed base-256 digits in [-128, 127])
constexpr int OZ_SA = 5;         // digit planes of an FP32 A (24-bit mantissas, 40 bits below the row scale)
#ifndef RSVD_OZ_SQ
#define RSVD_OZ_SQ 6
#endif
constexpr int OZ_SQ = RSVD_OZ_SQ;  // digit planes of an FP64 orthonormal basis: 6 = 48 bits below the column
                                 // scale (7 = 56 bits measured the same C2 parity, 1.995e-6 vs 1.998e-6, for
                                 // 14 % more plane bytes: C2 28.8 -> 28.4 ms with 6)
constexpr int OZ_LV_A = 6;       // A products: kept levels i + j <= 5, 6 B digits (20 pairs)
constexpr int OZ_LV_Q = 7;       // basis products: levels i + j <= 6, 7 B digits, 27 digit pairs (448 TMEM columns at BN 64)
constexpr int OZ_LV_R = 4;       // reduced A products (levels i + j <= 3, A digits 0..3, 10 pairs): ~1e-10
                                 // relative, for the Rayleigh-Ritz W = A^T Q (its error enters sigma^2
                                 // linearly, against the chain's 1e-15 amplified ~1e9 by the basis)
constexpr int OZ_SB_MAX = 7;
constexpr int OZ_STAGES = 5;
constexpr int64_t OZ_MAX_K = 16384;  // int32 exactness: 7 pairs x 128^2 x 16384 < 2^31
constexpr int OZ_THREADS = 10 * 32;  // 0 TMA, 1 MMA, 2..9 epilogue (two warps per TMEM lane quarter)
constexpr uint32_t kLayoutNone = 0;

// SA digit planes of the A operand, LV kept levels i + j < LV, as many B digits
template <int BN, int SA, int LV>
struct OzCfg {
    static constexpr int SB = LV;
    static constexpr int A_TILE = OZ_BM * OZ_KS;            // 4 KB per digit plane
    static constexpr int B_TILE = BN * OZ_KS;               // per digit plane
    static constexpr int STAGE = SA * A_TILE + SB * B_TILE;
    static constexpr int SMEM = OZ_STAGES * STAGE + 1024 + 256;
    static constexpr int ACC_COLS = LV * BN;
    static_assert(SMEM <= 227 * 1024, "stages do not fit shared memory");
    static_assert(ACC_COLS <= 512, "levels do not fit TMEM");
    static_assert(STAGE % 128 == 0, "stages must stay 128-byte aligned (TMA destinations; no swizzle is used)");
};

struct OzParams {
    int64_t M, N, K;         // D[M x N] = Aop[M x K] Bop[K x N]
    int64_t Np;              // rows per B digit plane
    const int8_t* a_planes;  // [SA][a_cols / 16][a_rows][16 B]
    int64_t a_rows;          // padded rows of A (multiple of 128)
    int64_t a_pitch;         // bytes per A plane
    const int8_t* b_planes;  // [K / 32][2][SB][Np][16 B]
    int64_t k_per_split;     // multiple of OZ_KS
    const int32_t* ea;       // per-M exponent (NN: A row exponents), nullptr for TN
    const int32_t* fb;       // per-N exponent of B's columns
    int direct;              // 1: C = alpha D + beta C (FP64); 0: FP64 partial to ws[z]
    double* C;
    int64_t ldc;
    double alpha, beta;
    double* ws;
    int64_t ldw;
    const int32_t* pred;
    int n_tiles, m_tiles, splits;
    int ablate;              // profiling ablations (RSVD_OZ_ABLATE): 1 no B loads, 2 no A loads, 4 no MMAs
};

// kind::i8 instruction descriptor: S32 accumulate, signed int8 A / B.
__host__ __device__ constexpr uint32_t oz_idesc(int M, int N, int a_mn_major) {
    return (2u << 4)                        // c_format S32
           | (1u << 7)                      // a_format signed 8 bit
           | (1u << 10)                     // b_format signed 8 bit
           | ((uint32_t)a_mn_major << 15)   // a major
           | ((uint32_t)(N >> 3) << 17)     // N
           | ((uint32_t)(M >> 4) << 24);    // M
}

__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld16_s32(uint32_t taddr, int32_t* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (int32_t)r[i];
}

#ifdef RSVD_OZ_TRACE
// clock64 / globaltimer stamps of the first 512 CTAs: start, after setup,
// acc_full seen, epilogue done (tools/oz_trace.py builds with -DRSVD_OZ_TRACE)
__device__ unsigned long long g_oz_trace[512][5];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define OZ_STAMP(i) do { if (blockIdx.x < 512 && blockIdx.z == 0) g_oz_trace[blockIdx.x][i] = gtime(); } while (0)
#else
#define OZ_STAMP(i) do { } while (0)
#endif

template <int BN, bool A_MN, int SA, int LV>
__global__ void __launch_bounds__(OZ_THREADS, 1)
k_oz_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, OzParams p) {
    if (pred_off(p.pred)) return;
    if (threadIdx.x == 0) OZ_STAMP(0);
    using Cfg = OzCfg<BN, SA, LV>;
    constexpr int SB = Cfg::SB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OZ_STAGES * Cfg::STAGE);
    uint64_t* full = bars;
    uint64_t* empty = bars + OZ_STAGES;
    uint64_t* acc_full = bars + 2 * OZ_STAGES;
    uint64_t* tmem_empty = bars + 2 * OZ_STAGES + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // Persistent CTA: work units (split z, M tile, N tile) are taken round-robin,
    // u = blockIdx.x, + gridDim.x, ... The producer runs ahead into the next
    // unit while the epilogue drains the accumulators (one CTA per unit left
    // the SM's loads idle for the epilogue, teardown, launch and setup of the
    // next CTA: ~10 us against a ~45 us main loop at C2, which capped the
    // plane stream at ~4.7 TB/s); the MMA issuer waits on tmem_empty, which the
    // epilogue warps release as soon as their levels are combined in registers.
    const int tiles = p.m_tiles * p.n_tiles;
    const int units = tiles * p.splits;
    auto unit_of = [&](int u, int64_t& m0, int64_t& n0, int& z, int64_t& kbeg, int& nks) {
        z = u / tiles;
        const int t = u - z * tiles;
        m0 = (int64_t)(t / p.n_tiles) * OZ_BM;
        n0 = (int64_t)(t % p.n_tiles) * BN;
        kbeg = (int64_t)z * p.k_per_split;
        const int64_t kend = min(p.K, kbeg + p.k_per_split);
        nks = kend > kbeg ? (int)((kend - kbeg + OZ_KS - 1) / OZ_KS) : 0;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < OZ_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(tmem_empty, OZ_THREADS / 32 - 2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        if (p.Np != BN) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
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
    if (threadIdx.x == 0) OZ_STAMP(1);

    if (warp == 0) {
        if (lane == 0) {  // ---------------- producer: 1-D bulk copies of contiguous runs
            // A planes [i][c / 16][r][16 B] (rows / columns zero-padded to multiples of
            // 128): NN tile = 2 runs of 128 rows x 16 B; TN tile = 8 runs of 32 rows x 16 B.
            // B planes [kb][half][j][c][16 B]: one run per (half, digit), or the whole
            // stage when a single N tile spans all Np rows.
            int s = 0;
            uint32_t ph = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int64_t m0, n0, kbeg;
                int z, nks;
                unit_of(u, m0, n0, z, kbeg, nks);
                for (int kb = 0; kb < nks; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    const int64_t kk = kbeg + (int64_t)kb * OZ_KS;
                    uint8_t* st = smem + s * Cfg::STAGE;
                    mbar_expect_tx(&full[s], Cfg::STAGE - ((p.ablate & 1) ? SB * Cfg::B_TILE : 0) -
                                                 ((p.ablate & 2) ? SA * Cfg::A_TILE : 0));
                    if (!(p.ablate & 2)) {
                        // all SA digit planes of the tile in ONE TMA box (u64 view of the 16-byte
                        // row pieces): NN 128 rows x 2 column blocks, TN 32 rows x 8 column blocks,
                        // landing as [plane][block][row][16 B]. (Per-plane bulk copies -- 13 to 15
                        // issues per K step from the one producer thread -- capped the short-K
                        // basis products at ~2 TB/s.)
                        if (!A_MN)
                            tma_load_3d(&tmA, &full[s], st, (int)(m0 * 2), (int)(kk / 16), 0);
                        else
                            tma_load_3d(&tmA, &full[s], st, (int)(kk * 2), (int)(m0 / 16), 0);
                    }
                    if (!(p.ablate & 1)) {
                        uint8_t* dst = st + SA * Cfg::A_TILE;
                        if (p.Np == BN)  // the whole stage is one contiguous run
                            bulk_g2s(dst, p.b_planes + (kk / OZ_KS) * 2 * SB * p.Np * 16, SB * Cfg::B_TILE,
                                     &full[s]);
                        else  // 2 SB runs of BN x 16 B: one TMA box
                            tma_load_3d(&tmB, &full[s], dst, (int)(n0 * 2), 0, (int)(kk / OZ_KS));
                    }
                    if (++s == OZ_STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            int s = 0;
            uint32_t ph = 0, tph = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int64_t m0, n0, kbeg;
                int z, nks;
                unit_of(u, m0, n0, z, kbeg, nks);
                if (nks == 0) continue;
                // the previous unit's accumulators have been read out
                mbar_wait(tmem_empty, tph ^ 1);
                tph ^= 1;
                tc_fence_after();
                for (int kb = 0; kb < nks; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * Cfg::STAGE);
                    const uint32_t bst = st + SA * Cfg::A_TILE;
#pragma unroll
                    for (int i = 0; i < SA; ++i) {
                        // no-swizzle core matrices (8 rows x 16 B, 128 contiguous bytes):
                        // K-major A [half][r][16 B]: 8-row groups SBO 128 B, K halves LBO 2 KB;
                        // MN-major A [mb][k][16 B]: 16-column blocks SBO 512 B, 8-row K groups LBO 128 B
                        const uint64_t da = A_MN ? make_desc(st + i * Cfg::A_TILE, 128, 512, kLayoutNone)
                                                 : make_desc(st + i * Cfg::A_TILE, 2048, 128, kLayoutNone);
                        const int nj = LV - i;  // B digits j with i + j < LV
                        const int rows = nj * BN;
#pragma unroll
                        for (int r0 = 0; r0 < SB * BN; r0 += 256) {
                            if (r0 >= rows) break;
                            // N is a multiple of 16 (M = 128): with BN = 56 an odd digit count
                            // rounds up by 8 columns, which land past the last level's columns
                            // (unused TMEM) and read 8 more rows of the B tile (the next digit)
                            const int nn = (rows - r0) < 256 ? ((rows - r0 + 15) & ~15) : 256;
                            // B [half][j][c][16 B]: rows j BN + c, 8-row groups SBO 128 B, halves LBO
                            const uint64_t db = make_desc(bst + r0 * 16, SB * BN * 16, 128, kLayoutNone);
                            const uint32_t acc = (kb == 0 && i == 0) ? 0u : 1u;
                            if (p.ablate & 4) continue;
                            tc_mma_i8(tmem_base + (uint32_t)(i * BN + r0), da, db, oz_idesc(OZ_BM, nn, A_MN ? 1 : 0),
                                      acc);
                        }
                    }
                    tc_commit(&empty[s]);
                    if (++s == OZ_STAGES) { s = 0; ph ^= 1; }
                }
                tc_commit(acc_full);
            }
        }
    } else {
        // ---------------- epilogue: thread = one output row (its TMEM lane)
        const int quarter = warp % 4;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        // two epilogue warps per lane quarter, each drains half of the columns
        const int half = (warp - 2) / 4;
        constexpr int HC = BN / 2;             // columns per epilogue thread
        constexpr int PC = HC > 32 ? 32 : HC;  // columns per pass (64 FP64 values in registers at most)
        constexpr int NPS = HC / PC;
        static_assert(NPS * PC == HC, "passes must tile the thread's columns");
        constexpr int NCH = (PC + 15) / 16;    // 16-column chunks per pass (the last one partly used when BN = 56)
        // per-column scale 2^(ea + fb - 16) as an exact power-of-two multiply
        // (ldexp's general path, 64 calls per thread, was a large part of a
        // ~20 us per-CTA epilogue), with ldexp kept for exponents outside the
        // normal range
        auto scale_of = [&](int e) -> double {
            return (e > -1022 && e < 1023) ? __longlong_as_double((long long)(e + 1023) << 52) : 0.0;
        };
        auto pow2 = [](int e) -> double { return __longlong_as_double((long long)(e + 1023) << 52); };
        constexpr int NG = (LV + 2) / 3;
        uint32_t aph = 0;
        bool first = true;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            int64_t m0, n0, kbeg;
            int z, nks;
            unit_of(u, m0, n0, z, kbeg, nks);
            const int64_t row = m0 + quarter * 32 + lane;
            if (p.direct && p.beta != 0.0 && row < p.M) {
                // C is read back by the epilogue (beta != 0): pull this thread's row
                // segment into L2 while the main loop runs
                for (int c = half * HC; c < (half + 1) * HC && n0 + c < p.N; c += 16)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(p.C + row * p.ldc + n0 + c));
            }
            int ea = 0;
            if (p.ea && row < p.M) ea = p.ea[row];
            // The epilogue is latency-bound (one warp per SM sub-partition): the
            // levels are combined in 64-bit integer arithmetic, three at a time --
            // g = acc_L 2^16 + acc_(L+1) 2^8 + acc_(L+2), below 2^48 so its conversion
            // is exact -- and the groups summed from the least significant up with
            // one FMA each: one int->FP64 conversion per three levels instead of
            // one per level (the Horner form made the epilogue ~14-16 us per CTA,
            // 20 % of a chain product). All of the thread's columns are combined
            // before anything is stored, so that TMEM goes back to the MMA issuer
            // after ~2 us and the stores overlap the next unit's main loop.
            // (BN = 128, the wide Rayleigh-Ritz product: two passes of 32 columns, TMEM
            // handed back after the second pass's loads)
            if (nks > 0) {
                mbar_wait(acc_full, aph);
                aph ^= 1;
                tc_fence_after();
                if (first && warp == 2 && lane == 0) OZ_STAMP(2);
            }
#pragma unroll
            for (int ps = 0; ps < NPS; ++ps) {
                const int pb = half * HC + ps * PC;  // first column of the pass
                double v[NCH][16];
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                    for (int t = 0; t < 16; ++t) v[ch][t] = 0.0;
                if (nks > 0) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) {
                        const int c0 = pb + ch * 16;
#pragma unroll
                        for (int g = NG - 1; g >= 0; --g) {
                            const int L0 = 3 * g;
                            const int L1 = L0 + 3 < LV ? L0 + 3 : LV;
                            int32_t a[3][16];
#pragma unroll
                            for (int L = 0; L < 3; ++L)
                                if (L0 + L < L1)
                                    tmem_ld16_s32(tmem_base + lane_off + (uint32_t)((L0 + L) * BN + c0), a[L]);
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                            const double wg = pow2(-OZ_DB * (L1 - 1));
#pragma unroll
                            for (int t = 0; t < 16; ++t) {
                                int64_t h = 0;
#pragma unroll
                                for (int L = 0; L < 3; ++L)
                                    if (L0 + L < L1) h = h * (1 << OZ_DB) + a[L][t];
                                v[ch][t] = fma((double)h, wg, v[ch][t]);
                            }
                        }
                    }
                    if (ps == NPS - 1) {
                        // accumulators read: hand TMEM back
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(tmem_empty);
                    }
                }
                // scale and store, 8 columns (64 bytes of the thread's row) at a time
#pragma unroll
                for (int c8 = 0; c8 < (PC + 7) / 8; ++c8) {
                    const int c0 = pb + c8 * 8;
                    const int left = HC - ps * PC - c8 * 8;
                    const int lim = left < 8 ? left : 8;  // columns of this thread's half in the chunk
                    const double* vv = &v[c8 / 2][(c8 % 2) * 8];
                    double sc[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const int64_t col = n0 + c0 + t;
                        sc[t] = (col < p.N && t < lim) ? scale_of(ea + p.fb[col] - 2 * OZ_DB) : 0.0;
                    }
                    if (row < p.M && n0 + c0 < p.N) {
                        const int64_t base =
                            p.direct ? row * p.ldc + n0 + c0 : ((int64_t)z * p.M + row) * p.ldw + n0 + c0;
                        double* out = p.direct ? p.C + base : p.ws + base;
                        const bool full8 =
                            lim == 8 && n0 + c0 + 8 <= p.N && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
                        // all loads of the chunk before any store (C is read and written)
                        double cin[8];
                        const bool rmw = p.direct && p.beta != 0.0;
                        if (rmw && full8) {
#pragma unroll
                            for (int t = 0; t < 8; t += 2) {
                                const double2 c2 = *reinterpret_cast<const double2*>(out + t);
                                cin[t] = c2.x;
                                cin[t + 1] = c2.y;
                            }
                        } else {
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                cin[t] = (rmw && t < lim && n0 + c0 + t < p.N) ? out[t] : 0.0;
                        }
                        double res[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const double val =
                                sc[t] != 0.0 ? vv[t] * sc[t]
                                             : ldexp(vv[t], ea + p.fb[min(n0 + c0 + t, p.N - 1)] - 2 * OZ_DB);
                            res[t] = p.direct ? (rmw ? p.alpha * val + p.beta * cin[t] : p.alpha * val) : val;
                        }
                        if (full8) {
#pragma unroll
                            for (int t = 0; t < 8; t += 2)
                                *reinterpret_cast<double2*>(out + t) = make_double2(res[t], res[t + 1]);
                        } else {
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                if (t < lim && n0 + c0 + t < p.N) out[t] = res[t];
                        }
                    }
                }
            }
            if (first && warp == 2 && lane == 0) OZ_STAMP(3);
            first = false;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
    if (threadIdx.x == 32) OZ_STAMP(4);
}

// ---------------------------------------------------------------- slicing
// Scale exponent of a row / column with maximum magnitude m > 0: the smallest
// E with m 2^-E <= 0.498, so that N = rint(x 2^(8 S - E)) has S signed
// base-256 digits in [-128, 127] (|N| <= 127 (256^S - 1) / 255 = 0.49804 256^S).
__device__ __forceinline__ int oz_exp_for(double m) {
    int e;
    const double f = frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
    const int E = f > 0.996 ? e + 2 : e + 1;
    return E < -960 ? -960 : E;  // keeps 2^(8 S - E) finite (columns below 1e-289 lose digits, not range)
}

// Signed base-256 digits of an integer N (least significant first: d = the
// sign-extended low byte, N = (N - d) / 256) are the bytes of (N + B) ^ B with
// B = 0x80...80: adding 128 at every digit position maps the digits to plain
// bytes, the XOR maps each byte back to two's complement. Digit i (0 = most
// significant of S) is byte S - 1 - i. Rounding x to the integer N first
// (round to nearest, zero-mean remainder) is what keeps every digit inside
// int8: rounding digit by digit from the top would need +128.
template <int S>
__device__ __forceinline__ unsigned long long oz_digits(long long N) {
    unsigned long long B = 0;
#pragma unroll
    for (int i = 0; i < S; ++i) B |= 0x80ull << (8 * i);
    return ((unsigned long long)N + B) ^ B;
}

__device__ __forceinline__ uint32_t oz_byte(unsigned long long M, int k) { return (uint32_t)(M >> (8 * k)) & 0xFFu; }

// Digit planes of A in the column-blocked layout planes[i][c / 16][r][c % 16]
// over n_pad x d_pad (both multiples of 128; padding written as zeros): a
// 16-byte row piece is one row of a tensor-core core matrix in either
// orientation. One CTA per 32 rows: warps find the row maxima (4 rows each),
// then lane l owns row r0 + l and each warp walks 16-column blocks, so a warp
// writes one contiguous 512-byte run per digit plane and block.
__global__ void __launch_bounds__(256) k_oz_slice_a(int64_t n, int64_t d, const float* __restrict__ A, int64_t lda,
                                                    int64_t n_pad, int64_t d_pad, int8_t* __restrict__ planes,
                                                    int32_t* __restrict__ row_exp, int64_t row0) {
    __shared__ double s_scale[32];
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
    const int64_t r0 = row0 + (int64_t)blockIdx.x * 32;
    const bool vec = (lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    for (int rr = warp; rr < 32; rr += 8) {
        const int64_t r = r0 + rr;
        float m = 0.f;
        if (r < n) {
            const float* a = A + r * lda;
            const int64_t d4 = vec ? d / 4 : 0;
            for (int64_t c = lane; c < d4; c += 32) {
                const float4 v = reinterpret_cast<const float4*>(a)[c];
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
            }
            for (int64_t c = d4 * 4 + lane; c < d; c += 32) m = fmaxf(m, fabsf(a[c]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const int E = m > 0.f ? oz_exp_for((double)m) : 0;
        if (lane == 0) {
            if (r < n) row_exp[r] = E;
            s_scale[rr] = ldexp(1.0, OZ_DB * OZ_SA - E);  // FP64: 2^(40 - E) overflows FP32 for tiny rows
        }
    }
    __syncthreads();
    const int64_t r = r0 + lane;
    const bool live = r < n;
    const double sc = s_scale[lane];
    const float* a = A + (live ? r : 0) * lda;
    const int64_t pp = n_pad * d_pad;  // plane pitch
    const bool vrow = vec && live;
    for (int64_t b = warp; b < d_pad / 16; b += 8) {
        float x[16];
        if (vrow && b * 16 + 16 <= d) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                const float4 v = reinterpret_cast<const float4*>(a + b * 16)[q4];
                x[4 * q4] = v.x; x[4 * q4 + 1] = v.y; x[4 * q4 + 2] = v.z; x[4 * q4 + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int t = 0; t < 16; ++t) x[t] = (live && b * 16 + t < d) ? a[b * 16 + t] : 0.f;
        }
        unsigned long long M[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) M[t] = oz_digits<OZ_SA>(__double2ll_rn((double)x[t] * sc));
        int8_t* out = planes + (b * n_pad + r) * 16;
#pragma unroll
        for (int i = 0; i < OZ_SA; ++i) {
            uint32_t w[4];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
                w[q4] = oz_byte(M[4 * q4], OZ_SA - 1 - i) | (oz_byte(M[4 * q4 + 1], OZ_SA - 1 - i) << 8) |
                        (oz_byte(M[4 * q4 + 2], OZ_SA - 1 - i) << 16) | (oz_byte(M[4 * q4 + 3], OZ_SA - 1 - i) << 24);
            *reinterpret_cast<uint4*>(out + i * pp) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

// Digit planes of columns [c0, c0 + ncols) of a basis Q (row pitch ldq), each
// column with its own exponent col_exp[c] (2^E > 2 max_r |Q[r, c]|): thread =
// one row of one 16-column block; bytes of columns outside the range are kept
// (read-modify-write of the 16-byte row piece), rows >= n written as zeros.
__global__ void __launch_bounds__(256) k_oz_slice_cols(int64_t n, const double* __restrict__ Q, int64_t ldq,
                                                       int64_t c0, int64_t ncols, int64_t n_pad, int64_t w_pad,
                                                       int8_t* __restrict__ planes, const int32_t* __restrict__ col_exp) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_pad) return;
    const int64_t b = c0 / 16 + blockIdx.y;
    const int64_t pp = n_pad * w_pad;
    unsigned long long M[16];
    bool mine[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        const int64_t c = b * 16 + t;
        mine[t] = c >= c0 && c < c0 + ncols;
        const double x = (mine[t] && r < n) ? ldexp(Q[r * ldq + c], OZ_DB * OZ_SQ - col_exp[c]) : 0.0;
        M[t] = oz_digits<OZ_SQ>(__double2ll_rn(x));
    }
#pragma unroll
    for (int i = 0; i < OZ_SQ; ++i) {
        uint4* dst = reinterpret_cast<uint4*>(planes + i * pp + (b * n_pad + r) * 16);
        uint4 old = *dst;
        uint32_t wv[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
        for (int t = 0; t < 16; ++t)
            if (mine[t]) {
                const int sh = (t % 4) * 8;
                wv[t / 4] = (wv[t / 4] & ~(0xFFu << sh)) | (oz_byte(M[t], OZ_SQ - 1 - i) << sh);
            }
        *dst = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
}

// B operand (K x N FP64, row pitch ldb), optional per-row exponent e_k folded
// in (A^T Y: Y[k, :] 2^E_k). Pass 1: per-column max of |2^e_k B[k, c]| as
// ordered bit patterns (atomicMax on the FP64 bits of a non-negative value).
__global__ void __launch_bounds__(256) k_oz_colmax_b(int64_t K, int64_t N, const double* __restrict__ B, int64_t ldb,
                                                     const int32_t* __restrict__ ek,
                                                     unsigned long long* __restrict__ colmax) {
    const int c = threadIdx.x % 32;  // 32 columns x 8 row groups per CTA
    const int g = threadIdx.x / 32;
    const int64_t col = (int64_t)blockIdx.y * 32 + c;
    double m = 0.0;
    if (col < N)
        for (int64_t k = (int64_t)blockIdx.x * 8 + g; k < K; k += (int64_t)gridDim.x * 8) {
            double v = fabs(B[k * ldb + col]);
            if (ek) v = ldexp(v, ek[k]);
            m = fmax(m, v);
        }
    __shared__ double red[8][32];
    red[g][c] = m;
    __syncthreads();
    if (g == 0 && col < N) {
#pragma unroll
        for (int i = 1; i < 8; ++i) m = fmax(m, red[i][c]);
        atomicMax(colmax + col, (unsigned long long)__double_as_longlong(m));
    }
}

__global__ void k_oz_col_exp(int64_t N, const unsigned long long* __restrict__ colmax, int32_t* __restrict__ fb) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    const double m = __longlong_as_double((long long)colmax[c]);
    fb[c] = m > 0.0 ? oz_exp_for(m) : 0;
}

// Pass 2: transposed digit planes in the k-blocked layout
// planes[k / 32][(k / 16) % 2][j][c][k % 16] (one K = 32 MMA step of all digits
// is one contiguous run; rows c in [N, Np) and k >= K written as zeros),
// through a 32 (k) x 32 (c) smem tile.
template <int SB>
__global__ void __launch_bounds__(256) k_oz_slice_b(int64_t K, int64_t N, const double* __restrict__ B, int64_t ldb,
                                                    const int32_t* __restrict__ ek,
                                                    const unsigned long long* __restrict__ colmax,
                                                    int32_t* __restrict__ fb,
                                                    int64_t Np, int64_t Kp, int8_t* __restrict__ planes) {
    __shared__ uint32_t tile[SB][32][9];  // [plane][c][k / 4] packed digits
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
    const int64_t k0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    // load: thread (tx = c, ty) handles rows k0 + 4 ty .. 4 ty + 3 of column c0 + tx
    const int64_t col = c0 + tx;
    // column exponent from the column maximum (pass 1); the k-block-0 CTAs
    // publish it for the GEMM epilogue
    int f = 0;
    if (col < N) {
        const double m = __longlong_as_double((long long)colmax[col]);
        f = m > 0.0 ? oz_exp_for(m) : 0;
        if (blockIdx.x == 0 && ty == 0) fb[col] = f;
    }
    const double sc = col < N ? ldexp(1.0, OZ_DB * SB - f) : 0.0;
    unsigned long long M[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int64_t k = k0 + 4 * ty + t;
        double u = 0.0;
        if (k < K && col < N) {
            u = B[k * ldb + col];
            if (ek) u = ldexp(u, ek[k]);
            u *= sc;
        }
        M[t] = oz_digits<SB>(__double2ll_rn(u));
    }
#pragma unroll
    for (int j = 0; j < SB; ++j)
        tile[j][tx][ty] = oz_byte(M[0], SB - 1 - j) | (oz_byte(M[1], SB - 1 - j) << 8) |
                          (oz_byte(M[2], SB - 1 - j) << 16) | (oz_byte(M[3], SB - 1 - j) << 24);
    __syncthreads();
    // store: rows c = c0 + (warp), 8 words of 4 k each per (plane, row)
    for (int e = threadIdx.x; e < SB * 32 * 8; e += blockDim.x) {
        const int w = e % 8, cc = (e / 8) % 32, j = e / 256;
        const int64_t c = c0 + cc;
        const int64_t k = k0 + 4 * w;
        if (c < Np)
            *reinterpret_cast<uint32_t*>(planes + ((((k0 / 32) * 2 + w / 4) * SB + j) * Np + c) * 16 + 4 * (w % 4)) =
                tile[j][cc][w];
    }
}

__global__ void k_oz_reduce(int64_t M, int64_t N, int64_t ldw, int64_t splits, const double* __restrict__ ws,
                            double alpha, double beta, double* __restrict__ C, int64_t ldc,
                            const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    const int64_t r = e / N, c = e % N;
    double v = 0.0;
    for (int64_t s = 0; s < splits; ++s) v += ws[(s * M + r) * ldw + c];
    v *= alpha;
    if (beta != 0.0) v += beta * C[r * ldc + c];
    C[r * ldc + c] = v;
}

// ---------------------------------------------------------------- host
// u64 views of the digit planes (a 16-byte row piece = 2 elements), no swizzle
// (the interleaved core-matrix layout is the gmem layout itself): one box =
// every used digit plane of a tile -- NN {128 rows, 2 column blocks, used},
// TN {32 rows, 8 column blocks, used}. B: u32 view, BN x 16 B rows.
int oz_map_a(CUtensorMap* map, const int8_t* planes, int64_t a_rows, int64_t d_pad, int64_t pitch, int nplanes,
             int used, bool mn_major) {
    EncodeTiledFn fn = encode_fn();
    RSVD_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {(cuuint64_t)(a_rows * 2), (cuuint64_t)(d_pad / 16), (cuuint64_t)nplanes};
    cuuint64_t strides[2] = {(cuuint64_t)(a_rows * 16), (cuuint64_t)pitch};
    cuuint32_t box[3] = {mn_major ? (cuuint32_t)(OZ_KS * 2) : (cuuint32_t)(OZ_BM * 2), mn_major ? 8u : 2u,
                         (cuuint32_t)used};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<int8_t*>(planes), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RSVD_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (Ozaki A planes) failed (%d)", (int)r);
    return RSVD_OK;
}

int oz_map_b(CUtensorMap* map, const int8_t* planes, int64_t Np, int64_t nkb, int bn, int sb) {
    EncodeTiledFn fn = encode_fn();
    RSVD_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
    // u64 view (a 16-byte row piece = 2 elements): the box's inner extent stays <= 256 at BN = 128
    cuuint64_t dims[3] = {(cuuint64_t)(Np * 2), (cuuint64_t)(2 * sb), (cuuint64_t)nkb};
    cuuint64_t strides[2] = {(cuuint64_t)(Np * 16), (cuuint64_t)(2 * sb * Np * 16)};
    cuuint32_t box[3] = {(cuuint32_t)(bn * 2), (cuuint32_t)(2 * sb), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<int8_t*>(planes), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RSVD_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (Ozaki B planes) failed (%d)", (int)r);
    return RSVD_OK;
}

// N tile: 56 for widths 33..56 (C2's p = 50: 12.5 % fewer MMA columns than 64; RSVD_OZ_BN56=0 keeps 64)
// Wide reduced products (the Rayleigh-Ritz W = A^T Q, 4 levels): 128, so that an
// A tile is streamed from L2 once per 128 output columns instead of once per 64
// (C2: the 10 N tiles of width 600 re-read the planes 10 x, 20 GB of L2 -> SM
// traffic in 2.26 ms; RSVD_OZ_BN128=0 keeps 64)
int oz_bn(int64_t n, bool reduced = false) {
    static const bool bn56 = !(getenv("RSVD_OZ_BN56") && atoi(getenv("RSVD_OZ_BN56")) == 0);
    static const bool bn128 = !(getenv("RSVD_OZ_BN128") && atoi(getenv("RSVD_OZ_BN128")) == 0);
    if (reduced && n > 64 && bn128) return 128;
    return n <= 32 ? 32 : (n <= 56 && bn56 ? 56 : 64);
}

// split count: K per CTA <= OZ_MAX_K (exactness), then the smallest count
// whose CTAs fill the SMs in waves >= 90% full (at most 64, >= 16 K steps
// each: a split's FP64 partials cost a write + read of the output, which a
// short reduction -- a projection against a 50..550-column prefix -- does
// not pay back)
int64_t oz_splits(int64_t tiles, int64_t K) {
    const int64_t min_s = cdiv(K, OZ_MAX_K);
    const int64_t G = sm_count();
    int64_t max_s = cdiv(K, 16 * OZ_KS);
    if (max_s > 64) max_s = 64;
    if (max_s < min_s) max_s = min_s;
    int64_t best = min_s;
    double best_e = 0.0;
    for (int64_t S = min_s; S <= max_s; ++S) {
        const double u = (double)(tiles * S) / (double)G;
        const double e = u / std::ceil(u);
        if (e > best_e + 1e-9) {
            best_e = e;
            best = S;
        }
        if (e >= 0.90) return S;
    }
    return best;
}

struct OzLayout {
    int bn;
    int64_t Np, Kp, splits, n_tiles, m_tiles;
    int64_t planes_off, colmax_off, fb_off, part_off, total;
};

OzLayout oz_layout(bool trans, int64_t n, int64_t d, int64_t p, bool reduced = false) {
    OzLayout L{};
    L.bn = oz_bn(p, reduced);
    const int64_t Mop = trans ? d : n, Kop = trans ? n : d;
    L.Np = cdiv(p, L.bn) * L.bn;
    L.Kp = cdiv(Kop, 32) * 32;
    L.n_tiles = cdiv(p, L.bn);
    L.m_tiles = cdiv(Mop, OZ_BM);
    L.splits = oz_splits(L.m_tiles * L.n_tiles, Kop);
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        int64_t o = off;
        off += cdiv(bytes, 256) * 256;
        return o;
    };
    L.planes_off = take((int64_t)OZ_SB_MAX * L.Np * L.Kp);
    L.colmax_off = take(p * 8);
    L.fb_off = take(p * 4);
    L.part_off = take(L.splits > 1 ? L.splits * Mop * p * 8 : 0);
    L.total = off + 256;
    return L;
}

template <int BN, bool A_MN, int SA, int LV>
int launch_oz(const CUtensorMap& tA, const CUtensorMap& tB, const OzParams& p, dim3 grid, cudaStream_t st) {
    using Cfg = OzCfg<BN, SA, LV>;
    static PerDevice<bool> attr_dev;
    bool& attr = attr_dev.get();
    if (!attr) {
        RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_oz_gemm<BN, A_MN, SA, LV>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
        attr = true;
    }
    k_oz_gemm<BN, A_MN, SA, LV><<<grid, OZ_THREADS, Cfg::SMEM, st>>>(tA, tB, p);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace

int64_t oz_planes_bytes(int64_t n, int64_t d) { return (int64_t)OZ_SA * cdiv(n, 128) * 128 * cdiv(d, 128) * 128; }
int oz_num_planes() { return OZ_SA; }

int oz_prepare(int64_t n, int64_t d, const float* A, int64_t lda, int8_t* planes, int32_t* row_exp,
               cudaStream_t st) {
    if (n == 0) return RSVD_OK;
    const int64_t n_pad = cdiv(n, 128) * 128, d_pad = cdiv(d, 128) * 128;
    k_oz_slice_a<<<(unsigned)(n_pad / 32), 256, 0, st>>>(n, d, A, lda, n_pad, d_pad, planes, row_exp, 0);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

// rows [r0, r0 + nr) of the n x d matrix A (r0 a multiple of 32): a row panel
// can be cut as soon as it has arrived in HBM, while the next panel's upload
// is still in flight; the panel that ends at row n also writes the zero
// padding rows up to the next multiple of 128.
int oz_prepare_rows(int64_t n, int64_t d, int64_t r0, int64_t nr, const float* A, int64_t lda, int8_t* planes,
                    int32_t* row_exp, cudaStream_t st) {
    RSVD_REQUIRE(r0 >= 0 && nr >= 0 && r0 + nr <= n && r0 % 32 == 0, "oz_prepare_rows: bad row range");
    if (nr == 0) return RSVD_OK;
    const int64_t n_pad = cdiv(n, 128) * 128, d_pad = cdiv(d, 128) * 128;
    const int64_t end = r0 + nr == n ? n_pad : r0 + nr;
    k_oz_slice_a<<<(unsigned)cdiv(end - r0, 32), 256, 0, st>>>(n, d, A, lda, n_pad, d_pad, planes, row_exp, r0);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int64_t oz_gemm_ws_bytes(int trans, int64_t n, int64_t d, int64_t p) {
    // covers the reduced (wide N tile) layout of the same product too
    return std::max(oz_layout(trans != 0, n, d, p, false).total, oz_layout(trans != 0, n, d, p, true).total);
}

// trans = 0: C (n x p) = alpha A X + beta C, X d x p.
// trans = 1: C (d x p) = alpha A^T Y + beta C, Y n x p.
// A is given by `nplanes` digit planes [i][c / 16][r][16 B] allocated for
// rows_alloc x cols_alloc (multiples of 128) and per-row exponents; the
// product uses its leading n x d corner (an orthonormal basis' prefix).
int oz_gemm_planes(int trans, int64_t n, int64_t d, int64_t p, double alpha, const int8_t* planes, int nplanes,
                   int64_t rows_alloc, int64_t cols_alloc, const int32_t* exps, int col_scaled, const double* B,
                   int64_t ldb, double beta, double* C, int64_t ldc, void* ws, int64_t ws_bytes, const int32_t* pred,
                   cudaStream_t st, int reduced) {
    const bool tr = trans != 0;
    RSVD_REQUIRE(!reduced || nplanes == OZ_SA, "oz_gemm: reduced accuracy is for the A planes");
    // exponents of the contraction index are folded into B before slicing it;
    // exponents of the output-row index scale the epilogue
    const bool fold = tr != (col_scaled != 0);
    RSVD_REQUIRE(nplanes == OZ_SA || nplanes == OZ_SQ, "oz_gemm: %d digit planes not supported", nplanes);
    RSVD_REQUIRE(rows_alloc % 128 == 0 && cols_alloc % 128 == 0 && rows_alloc >= n && cols_alloc >= d,
                 "oz_gemm: plane geometry does not cover the product");
    const OzLayout L = oz_layout(tr, n, d, p, reduced != 0);
    RSVD_REQUIRE(ws_bytes >= L.total, "oz_gemm: workspace too small (%lld < %lld)", (long long)ws_bytes,
                 (long long)L.total);
    RSVD_REQUIRE((reinterpret_cast<uintptr_t>(planes) & 15) == 0, "oz_gemm: digit planes must be 16-byte aligned");
    const int64_t Mop = tr ? d : n, Kop = tr ? n : d;
    if (Mop == 0 || p == 0) return RSVD_OK;
    uint8_t* w = reinterpret_cast<uint8_t*>(ws);
    int8_t* bpl = reinterpret_cast<int8_t*>(w + L.planes_off);
    unsigned long long* cmax = reinterpret_cast<unsigned long long*>(w + L.colmax_off);
    int32_t* fb = reinterpret_cast<int32_t*>(w + L.fb_off);
    double* part = reinterpret_cast<double*>(w + L.part_off);
    const int32_t* ek = fold ? exps : nullptr;
    RSVD_CHECK_CUDA(cudaMemsetAsync(cmax, 0, p * 8, st));
    {
        dim3 g((unsigned)std::min<int64_t>(cdiv(Kop, 8), 2 * sm_count()), (unsigned)cdiv(p, 32));
        k_oz_colmax_b<<<g, 256, 0, st>>>(Kop, p, B, ldb, ek, cmax);
        dim3 g2((unsigned)cdiv(L.Kp, 32), (unsigned)cdiv(L.Np, 32));
        if (reduced)
            k_oz_slice_b<OZ_LV_R><<<g2, 256, 0, st>>>(Kop, p, B, ldb, ek, cmax, fb, L.Np, L.Kp, bpl);
        else if (nplanes == OZ_SA)
            k_oz_slice_b<OZ_LV_A><<<g2, 256, 0, st>>>(Kop, p, B, ldb, ek, cmax, fb, L.Np, L.Kp, bpl);
        else
            k_oz_slice_b<OZ_LV_Q><<<g2, 256, 0, st>>>(Kop, p, B, ldb, ek, cmax, fb, L.Np, L.Kp, bpl);
        RSVD_CHECK_LAUNCH();
    }
    const int sb = reduced ? OZ_LV_R : (nplanes == OZ_SA ? OZ_LV_A : OZ_LV_Q);
    int rc = RSVD_OK;
    OzParams prm{};
    prm.a_planes = planes;
    prm.a_rows = rows_alloc;
    prm.a_pitch = rows_alloc * cols_alloc;
    prm.b_planes = bpl;
    CUtensorMap tA{}, tB{};
    rc = oz_map_a(&tA, planes, rows_alloc, cols_alloc, prm.a_pitch, nplanes,
                  reduced ? OZ_LV_R : nplanes, tr);
    if (rc) return rc;
    if (L.Np != L.bn) {
        rc = oz_map_b(&tB, bpl, L.Np, L.Kp / 32, L.bn, sb);
        if (rc) return rc;
    }
    prm.M = Mop; prm.N = p; prm.K = Kop; prm.Np = L.Np;
    prm.k_per_split = cdiv(cdiv(Kop, L.splits), OZ_KS) * OZ_KS;
    prm.ea = fold ? nullptr : exps;
    prm.fb = fb;
    prm.direct = L.splits == 1;
    prm.C = C; prm.ldc = ldc; prm.alpha = alpha; prm.beta = beta;
    prm.ws = part; prm.ldw = p;
    prm.pred = pred;
    prm.n_tiles = (int)L.n_tiles;
    prm.m_tiles = (int)L.m_tiles;
    prm.splits = (int)L.splits;
    {
        static const char* ab = getenv("RSVD_OZ_ABLATE");
        prm.ablate = ab ? atoi(ab) : 0;
    }
    // persistent CTAs, one per SM, over the (split, tile) work units
    dim3 grid((unsigned)std::min<int64_t>(L.m_tiles * L.n_tiles * L.splits, sm_count()), 1, 1);
#define RSVD_OZ_LAUNCH(SA_, LV_)                                                                         \
    do {                                                                                                 \
        if (L.bn == 32)                                                                                  \
            rc = tr ? launch_oz<32, true, SA_, LV_>(tA, tB, prm, grid, st)                               \
                    : launch_oz<32, false, SA_, LV_>(tA, tB, prm, grid, st);                             \
        else if (L.bn == 56)                                                                             \
            rc = tr ? launch_oz<56, true, SA_, LV_>(tA, tB, prm, grid, st)                               \
                    : launch_oz<56, false, SA_, LV_>(tA, tB, prm, grid, st);                             \
        else                                                                                             \
            rc = tr ? launch_oz<64, true, SA_, LV_>(tA, tB, prm, grid, st)                               \
                    : launch_oz<64, false, SA_, LV_>(tA, tB, prm, grid, st);                             \
    } while (0)
    if (reduced && L.bn == 128)
        rc = tr ? launch_oz<128, true, OZ_LV_R, OZ_LV_R>(tA, tB, prm, grid, st)
                : launch_oz<128, false, OZ_LV_R, OZ_LV_R>(tA, tB, prm, grid, st);
    else if (reduced)
        RSVD_OZ_LAUNCH(OZ_LV_R, OZ_LV_R);
    else if (nplanes == OZ_SA)
        RSVD_OZ_LAUNCH(OZ_SA, OZ_LV_A);
    else
        RSVD_OZ_LAUNCH(OZ_SQ, OZ_LV_Q);
#undef RSVD_OZ_LAUNCH
    if (rc) return rc;
    if (L.splits > 1) {
        const int64_t tot = Mop * p;
        k_oz_reduce<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(Mop, p, p, L.splits, part, alpha, beta, C, ldc, pred);
        RSVD_CHECK_LAUNCH();
    }
    return RSVD_OK;
}

int oz_gemm(int trans, int64_t n, int64_t d, int64_t p, double alpha, const int8_t* planes,
            const int32_t* row_exp, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* ws,
            int64_t ws_bytes, const int32_t* pred, cudaStream_t st) {
    return oz_gemm_planes(trans & 1, n, d, p, alpha, planes, OZ_SA, cdiv(n, 128) * 128, cdiv(d, 128) * 128, row_exp,
                          0, B, ldb, beta, C, ldc, ws, ws_bytes, pred, st, (trans & 2) != 0);
}

// ---- FP64 basis (n x w): OZ_SQ digit planes with per-COLUMN exponents
// (col_exp[w]), filled one block of columns at a time as the blocks become
// final. Column scaling makes both products exact-scaled: Q_p^T V scales its
// output rows by col_exp, Q_p C folds col_exp into C's rows (the contraction
// index), mirroring the row-scaled A planes.
int oz_basis_planes() { return OZ_SQ; }
int64_t oz_basis_bytes(int64_t n, int64_t w) { return (int64_t)OZ_SQ * cdiv(n, 128) * 128 * cdiv(w, 128) * 128; }

int64_t oz_basis_ws_bytes(int64_t ncols) { return ncols * 8 + 256; }

int oz_basis_slice(int64_t n, int64_t w, const double* Q, int64_t ldq, int64_t c0, int64_t ncols, int8_t* planes,
                   int32_t* col_exp, void* ws, int64_t ws_bytes, cudaStream_t st) {
    RSVD_REQUIRE(c0 >= 0 && ncols >= 0 && c0 + ncols <= w, "oz_basis_slice: column range outside the basis");
    RSVD_REQUIRE(ws_bytes >= oz_basis_ws_bytes(ncols), "oz_basis_slice: workspace too small");
    if (n == 0 || ncols == 0) return RSVD_OK;
    const int64_t n_pad = cdiv(n, 128) * 128, w_pad = cdiv(w, 128) * 128;
    unsigned long long* cmax = reinterpret_cast<unsigned long long*>(ws);
    RSVD_CHECK_CUDA(cudaMemsetAsync(cmax, 0, ncols * 8, st));
    dim3 g0((unsigned)std::min<int64_t>(cdiv(n, 8), 2 * sm_count()), (unsigned)cdiv(ncols, 32));
    k_oz_colmax_b<<<g0, 256, 0, st>>>(n, ncols, Q + c0, ldq, nullptr, cmax);
    k_oz_col_exp<<<(unsigned)cdiv(ncols, 128), 128, 0, st>>>(ncols, cmax, col_exp + c0);
    const int64_t b0 = c0 / 16, b1 = cdiv(c0 + ncols, 16);
    dim3 g((unsigned)cdiv(n_pad, 256), (unsigned)(b1 - b0));
    k_oz_slice_cols<<<g, 256, 0, st>>>(n, Q, ldq, c0, ncols, n_pad, w_pad, planes, col_exp);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace rsvd

#ifdef RSVD_OZ_TRACE
extern "C" int rsvd_debug_oz_trace(unsigned long long* host_out) {
    return (int)cudaMemcpyFromSymbol(host_out, rsvd::g_oz_trace, sizeof(rsvd::g_oz_trace));
}
#endif
