// tcgen05 3xTF32 tall-skinny GEMMs for the FP32 path (sm_100a).
//
//   NN:  C[m x n]  = alpha (A[m x k] B[k x n] - 1 row_sub^T) + beta C
//        operand A = A (K-major), operand B = B (MN-major), K = k
//   TN:  C[k x n]  = alpha (A^T B - mu colsum^T) + beta C   (reduction over m)
//        operand A = A^T (MN-major: A's columns are contiguous), operand B = B
//        (MN-major), K = m, split over K with FP64 reduction of the partials.
//
// FP32 accuracy from TF32 tensor cores by the hi/lo split
//   a = a_hi + a_lo, b = b_hi + b_lo  (hi = top 10 mantissa bits, exact in
//   TF32; lo = rna_tf32(x - hi)),   a b ~= a_hi b_hi + a_hi b_lo + a_lo b_hi.
// B (the small d x p / n x p block) is split once into a [hi; lo] array in
// global memory by k_split_b; A (the large matrix) is split on the fly:
//   TMA (SWIZZLE_128B) -> smem A stage -> 4 converter warps mask A_hi in
//   place and write A_lo to a sibling buffer -> fence.proxy.async -> one
//   elected thread issues 3 tcgen05.mma.kind::tf32 per K=8 step with the
//   FP32 accumulators in TMEM: D0 += A_hi B_hi, D1 += A_hi B_lo,
//   D0 += A_lo B_hi -> the epilogue warps tcgen05.ld D0 + D1.
// The TF32 tensor-core accumulator rounds with a bias (error measured to
// grow linearly in K: 4e-7 at K=32, 5e-6 at 1e3, 5e-5 at 1e4), so TMEM only
// accumulates KCHUNK = 4 k-blocks (K = 128); two accumulator sets alternate
// and four dedicated warps drain each finished chunk into round-to-nearest
// FP32 registers while the tensor core fills the other set.
// Warp roles (448 threads): w0 TMA producer, w1 MMA issuer (+TMEM alloc),
// w2..w9 converters, w10..w13 accumulator drain + epilogue (w % 4 covers the
// four TMEM lane quarters).
// Pipelines: full[s] (TMA bytes landed), conv[s] (A split ready), empty[s]
// (MMA done reading the stage, via tcgen05.commit), acc_full[2] / acc_empty[2]
// (TMEM accumulator sets).
#include <cuda.h>

#include "gemm.cuh"

namespace rsvd {

namespace {

constexpr int BM = 128;      // UMMA M
constexpr int BK = 32;       // fp32 elements per 128-byte swizzle row
constexpr int kConvWarps = 4;
constexpr int kConvThreads = 32 * kConvWarps;
constexpr int kDrainWarp0 = 2 + kConvWarps;      // first accumulator-drain warp
constexpr int kThreads = 32 * (kDrainWarp0 + 4);
constexpr int KCHUNK = 4;  // k-blocks accumulated in TMEM before a drain

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %0;" ::"r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// A operand from TMEM (lane = row, one 32-bit column per k), B from smem.
__device__ __forceinline__ void tc_mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor (sm_100, version 1).
//  K-major operands: SWIZZLE_128B (layout 2, 16-byte swizzle atoms, 8-row
//    groups, SBO = 1024 B), K advanced by 32 bytes per K=8 step.
//  MN-major 32-bit operands: SWIZZLE_128B_BASE32B (layout 1 = CuTe
//    Swizzle<2,5,2>: 32-byte chunks XOR (row % 4), 4-row K groups, SBO = 512
//    B, LBO = stride between 32-element MN atoms), K advanced by 8 rows =
//    1024 B per step. TMA writes this layout with SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    d |= (uint64_t)layout << 61;
    return d;
}
constexpr uint32_t kLayoutSW128 = 2, kLayoutSW128Base32 = 1;

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

// ------------------------------------------------------------------ kernel
struct TcParams {
    int64_t M, N, K;        // operand shapes: D[M x N] = Aop[M x K] Bop[K x N]
    int64_t k_per_split;    // K range per blockIdx.z (multiple of BK)
    int64_t Kp;             // padded K of the split-B array (rows of hi; lo starts at Kp)
    // epilogue
    int direct;             // 1: write C (NN); 0: FP32 partial to ws[z][M][N]
    float* C;
    int64_t ldc;
    double alpha, beta;
    const double* row_sub;
    float* ws;
    const int32_t* pred;
};

template <int BN, bool A_MN>
struct TcCfg {
    // A_lo in TMEM (tcgen05.mma .ts form) when the accumulators leave room:
    // the smem stage then holds only raw A (the tensor core truncates FP32 to
    // TF32 itself, so raw A *is* A_hi) and B_hi/B_lo -> deeper pipelines.
    static constexpr bool LO_TMEM = BN <= 64;
    static constexpr int BNP = ((BN + 31) / 32) * 32;  // B tile padded to whole 32-wide atoms
    static constexpr int A_BYTES = BM * BK * 4;         // 16 KB
    static constexpr int B_BYTES = BNP * BK * 4;
    static constexpr int STAGE_BYTES = (LO_TMEM ? 1 : 2) * A_BYTES + 2 * B_BYTES;
    static constexpr int ACC_COLS = 4 * BN;                 // 2 sets x (D0 | D1)
    static constexpr int STAGES_SMEM = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES_TMEM = LO_TMEM ? (512 - ACC_COLS) / BK : 64;
    static constexpr int STAGES_RAW = STAGES_SMEM < STAGES_TMEM ? STAGES_SMEM : STAGES_TMEM;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int TMEM_NEED = ACC_COLS + (LO_TMEM ? STAGES * BK : 0);
    static constexpr int TMEM_COLS = TMEM_NEED <= 128 ? 128 : (TMEM_NEED <= 256 ? 256 : 512);
    static constexpr int ALO_COL = ACC_COLS;  // first TMEM column of the A_lo stages
};

template <int BN, bool A_MN>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
    if (pred_off(p.pred)) return;
    using Cfg = TcCfg<BN, A_MN>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* full = bars;
    uint64_t* conv = bars + STAGES;
    uint64_t* empty = bars + 2 * STAGES;
    uint64_t* acc_full = bars + 3 * STAGES;   // [2]
    uint64_t* acc_empty = bars + 3 * STAGES + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int64_t n0 = (int64_t)blockIdx.y * BN;
    const int64_t kbeg = (int64_t)blockIdx.z * p.k_per_split;
    const int64_t kend = min(p.K, kbeg + p.k_per_split);
    const int nkb = (int)((kend - kbeg + BK - 1) / BK);

    auto a_stage = [&](int s) { return smem + s * Cfg::STAGE_BYTES; };
    auto alo_stage = [&](int s) { return smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES; };
    constexpr int kABufs = Cfg::LO_TMEM ? 1 : 2;  // [A | (A_lo) | B_hi | B_lo] per stage
    auto bhi_stage = [&](int s) { return smem + s * Cfg::STAGE_BYTES + kABufs * Cfg::A_BYTES; };
    auto blo_stage = [&](int s) { return smem + s * Cfg::STAGE_BYTES + kABufs * Cfg::A_BYTES + Cfg::B_BYTES; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], kConvWarps);
            mbar_init(&empty[s], 1);
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
                     "r"(Cfg::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&empty[s], ph ^ 1);
                const int kk = (int)(kbeg + (int64_t)kb * BK);
                mbar_expect_tx(&full[s], Cfg::A_BYTES + 2 * Cfg::B_BYTES);
                if (!A_MN) {
                    tma_load_2d(&tmA, &full[s], a_stage(s), kk, (int)m0);
                } else {
#pragma unroll
                    for (int i = 0; i < BM / 32; ++i)
                        tma_load_2d(&tmA, &full[s], a_stage(s) + i * 32 * BK * 4, (int)(m0 + 32 * i), kk);
                }
#pragma unroll
                for (int i = 0; i < Cfg::BNP / 32; ++i) {
                    tma_load_2d(&tmB, &full[s], bhi_stage(s) + i * 32 * BK * 4, (int)(n0 + 32 * i), kk);
                    tma_load_2d(&tmB, &full[s], blo_stage(s) + i * 32 * BK * 4, (int)(n0 + 32 * i),
                                (int)(p.Kp + kk));
                }
                if (++s == STAGES) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = make_idesc(BM, BN, A_MN ? 1 : 0, 1);
        constexpr uint32_t idesc_t = make_idesc(BM, BN, 0, 1);  // A_lo from TMEM
        int s = 0;
        uint32_t ph = 0;
        int chunk = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            const int set = chunk & 1;
            const uint32_t d0 = tmem_base + set * 2 * BN;
            if (kb % KCHUNK == 0) {
                mbar_wait(&acc_empty[set], ((chunk >> 1) & 1) ^ 1);
                tc_fence_after();
            }
            mbar_wait(&conv[s], ph);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t a_hi = smem_u32(a_stage(s));
                const uint32_t a_lo = Cfg::LO_TMEM ? 0u : smem_u32(alo_stage(s));
                const uint32_t b_hi = smem_u32(bhi_stage(s)), b_lo = smem_u32(blo_stage(s));
#pragma unroll
                for (int ks = 0; ks < BK / 8; ++ks) {
                    uint64_t da_hi, da_lo;
                    if (!A_MN) {  // K-major: advance 32 bytes inside the 128B row
                        da_hi = make_desc(a_hi + ks * 32, 16, 1024, kLayoutSW128);
                        da_lo = make_desc(a_lo + ks * 32, 16, 1024, kLayoutSW128);
                    } else {  // MN-major: advance 8 K rows
                        da_hi = make_desc(a_hi + ks * 1024, 32 * BK * 4, 512, kLayoutSW128Base32);
                        da_lo = make_desc(a_lo + ks * 1024, 32 * BK * 4, 512, kLayoutSW128Base32);
                    }
                    const uint64_t db_hi = make_desc(b_hi + ks * 1024, 32 * BK * 4, 512, kLayoutSW128Base32);
                    const uint64_t db_lo = make_desc(b_lo + ks * 1024, 32 * BK * 4, 512, kLayoutSW128Base32);
                    const uint32_t acc = (kb % KCHUNK > 0 || ks > 0) ? 1u : 0u;
                    tc_mma_tf32(d0, da_hi, db_hi, idesc, acc);
                    tc_mma_tf32(d0 + BN, da_hi, db_lo, idesc, acc);
                    if (Cfg::LO_TMEM)
                        tc_mma_tf32_ts(d0, tmem_base + Cfg::ALO_COL + s * BK + ks * 8, db_hi, idesc_t, 1u);
                    else
                        tc_mma_tf32(d0, da_lo, db_hi, idesc, 1u);
                }
                tc_commit(&empty[s]);
                if (kb % KCHUNK == KCHUNK - 1 || kb == nkb - 1) tc_commit(&acc_full[set]);
            }
            __syncwarp();
            if (kb % KCHUNK == KCHUNK - 1 || kb == nkb - 1) ++chunk;
            if (++s == STAGES) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp < kDrainWarp0) {
        if constexpr (Cfg::LO_TMEM) {
            // ---------------- converters: A_lo = rna(A - trunc(A)) straight into TMEM.
            // Thread (quarter q = warp % 4, lane l) owns tile row m = 32q + l, i.e.
            // its own TMEM lane, and converts the row's 32 k values in two halves.
            const int quarter = warp % 4;
            const int m = quarter * 32 + lane;
            const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full[s], ph);
                const uint8_t* a = a_stage(s);
#pragma unroll
                for (int kh = 0; kh < 2; ++kh) {
                float lo[16];
                if (!A_MN) {
                    // K-major SWIZZLE_128B: row m = 128 bytes, 16B chunk c at c ^ (m % 8)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int chunk = kh * 4 + c;
                        const float4 x = *reinterpret_cast<const float4*>(a + m * 128 + ((chunk ^ (m & 7)) << 4));
                        lo[4 * c + 0] = tf32_rna(x.x - tf32_hi(x.x));
                        lo[4 * c + 1] = tf32_rna(x.y - tf32_hi(x.y));
                        lo[4 * c + 2] = tf32_rna(x.z - tf32_hi(x.z));
                        lo[4 * c + 3] = tf32_rna(x.w - tf32_hi(x.w));
                    }
                } else {
                    // MN-major SWIZZLE_128B_BASE32B: atom q (32 M x 32 K) at q*4096,
                    // K row k = 128 bytes, 32B chunk (l/8) at (l/8) ^ (k % 4)
                    const uint8_t* atom = a + quarter * 4096 + (lane & 7) * 4;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int k = kh * 16 + i;
                        const float x = *reinterpret_cast<const float*>(atom + k * 128 + (((lane >> 3) ^ (k & 3)) << 5));
                        lo[i] = tf32_rna(x - tf32_hi(x));
                    }
                }
                tmem_st16(tmem_base + lane_off + Cfg::ALO_COL + s * BK + kh * 16, lo);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&conv[s]);
                if (++s == STAGES) {
                    s = 0;
                    ph ^= 1;
                }
            }
        } else {
        // ---------------- converters: A_hi in place, A_lo to the sibling buffer
        // (all loads of a thread's share first, then the split, then the stores)
        const int ct = threadIdx.x - 64;
        constexpr int PER = Cfg::A_BYTES / 16 / kConvThreads;
        int s = 0;
        uint32_t ph = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&full[s], ph);
            float4* a = reinterpret_cast<float4*>(a_stage(s));
            float4* lo = reinterpret_cast<float4*>(alo_stage(s));
            float4 xs[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) xs[i] = a[ct + i * kConvThreads];
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const float4 x = xs[i];
                const float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
                const float4 l = make_float4(tf32_rna(x.x - h.x), tf32_rna(x.y - h.y), tf32_rna(x.z - h.z),
                                             tf32_rna(x.w - h.w));
                a[ct + i * kConvThreads] = h;
                lo[ct + i * kConvThreads] = l;
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[s]);
            if (++s == STAGES) {
                s = 0;
                ph ^= 1;
            }
        }
        }
    } else {
        // ---------------- accumulator drain + epilogue; TMEM lanes 32*(warp%4)+lane = tile row
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
            const uint32_t base = tmem_base + lane_off + set * 2 * BN;
#pragma unroll
            for (int j = 0; j < BN; j += 8) {
                float v0[8], v1[8];
                tmem_ld8(base + j, v0);
                tmem_ld8(base + BN + j, v1);
#pragma unroll
                for (int i = 0; i < 8; ++i) sum[j + i] += v0[i] + v1[i];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[set]);
        }
        if (row < p.M) {
#pragma unroll
            for (int i = 0; i < BN; ++i) {
                const int64_t col = n0 + i;
                if (col < p.N) {
                    if (p.direct) {
                        double r = (double)sum[i];
                        if (p.row_sub) r -= p.row_sub[col];
                        r *= p.alpha;
                        if (p.beta != 0.0) r += p.beta * (double)p.C[row * p.ldc + col];
                        p.C[row * p.ldc + col] = (float)r;
                    } else {
                        p.ws[((int64_t)blockIdx.z * p.M + row) * p.N + col] = sum[i];
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS));
    }
}

// Split the small operand B (K x N, ld) into [hi; lo] rows of a (2 Kp) x Np
// array with zero padding (so TMA boxes past K or N read zeros).
__global__ void k_split_b(int64_t K, int64_t N, const float* __restrict__ B, int64_t ldb, int64_t Kp, int64_t Np,
                          float* __restrict__ out, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= Kp * Np) return;
    int64_t r = e / Np, c = e % Np;
    float x = (r < K && c < N) ? B[r * ldb + c] : 0.f;
    float h = tf32_hi(x);
    out[e] = h;
    out[Kp * Np + e] = tf32_rna(x - h);
}

template <typename TO>
__global__ void k_tc_reduce(int64_t M, int64_t N, int64_t splits, const float* __restrict__ ws, double alpha,
                            double beta, TO* __restrict__ C, int64_t ldc, const double* __restrict__ mu,
                            const double* __restrict__ cs, const int32_t* __restrict__ pred) {
    if (pred_off(pred)) return;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    int64_t r = e / N, c = e % N;
    double v = 0.0;
    for (int64_t s = 0; s < splits; ++s) v += (double)ws[s * M * N + e];
    if (mu) v -= mu[r] * cs[c];
    v *= alpha;
    if (beta != 0.0) v += beta * (double)C[r * ldc + c];
    C[r * ldc + c] = (TO)v;
}

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

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

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int pick_bn(int64_t n) {
    // widest tile first; the kernel is instantiated for these widths
    if (n <= 32) return 32;
    if (n <= 64) return 64;
    if (n <= 96) return 96;
    return 128;
}

template <int BN, bool A_MN>
int launch_tc(const CUtensorMap& tA, const CUtensorMap& tB, const TcParams& p, dim3 grid, cudaStream_t st) {
    using Cfg = TcCfg<BN, A_MN>;
    static bool attr_set = false;
    if (!attr_set) {
        RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_tc_gemm<BN, A_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Cfg::SMEM));
        attr_set = true;
    }
    k_tc_gemm<BN, A_MN><<<grid, kThreads, Cfg::SMEM, st>>>(tA, tB, p);
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
        default: return launch_tc<128, A_MN>(tA, tB, p, grid, st);
    }
}

// scratch for the split B array (grows; stream-ordered reuse)
struct Scratch {
    void* ptr = nullptr;
    size_t bytes = 0;
};

int split_b(const float* B, int64_t K, int64_t N, int64_t ldb, int64_t Kp, int64_t Np, float* out,
            const int32_t* pred, cudaStream_t st) {
    int64_t tot = Kp * Np;
    k_split_b<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(K, N, B, ldb, Kp, Np, out, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int64_t tn_splits_tc(int64_t Mop, int64_t Nop, int64_t Kop) {
    // split-K only for parallelism (accuracy is handled by the chunked TMEM
    // accumulation): enough CTAs to fill the chip, but few enough partials
    // that the reduction stays short.
    int bn = pick_bn(Nop);
    int64_t tiles = cdiv(Mop, BM) * cdiv(Nop, bn);
    int64_t target = (int64_t)sm_count() * 2;
    int64_t s = cdiv(target, tiles);
    if (s > 64) s = 64;
    int64_t max_s = cdiv(Kop, 8 * BK);
    if (s > max_s) s = max_s;
    if (s < 1) s = 1;
    return s;
}

}  // namespace

bool gemm_tc_nn_supported(int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc, const void* A,
                          const void* B) {
    (void)ldb; (void)ldc; (void)B;
    if (getenv("RSVD_DISABLE_TC")) return false;
    return m >= BM && k >= BK && n >= 1 && (lda % 4) == 0 && aligned16(A) && m < (1ll << 31) && k < (1ll << 31);
}

int gemm_nn_tc(int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda, const float* B,
               int64_t ldb, double beta, float* C, int64_t ldc, const double* row_sub, const int32_t* pred,
               cudaStream_t st) {
    int bn = pick_bn(n);
    const int64_t Kp = cdiv(k, BK) * BK, Np = cdiv(n, 32) * 32 + 128;
    static thread_local Scratch sc;  // split-B buffer
    size_t need = (size_t)(2 * Kp * Np * 4);
    if (sc.bytes < need) {
        if (sc.ptr) cudaFreeAsync(sc.ptr, st);
        RSVD_CHECK_CUDA(cudaMallocAsync(&sc.ptr, need, st));
        sc.bytes = need;
    }
    float* bs = (float*)sc.ptr;
    int rc = split_b(B, k, n, ldb, Kp, Np, bs, pred, st);
    if (rc) return rc;
    CUtensorMap tA, tB;
    rc = make_map(&tA, A, k, m, lda, BM, false);
    if (rc) return rc;
    rc = make_map(&tB, bs, Np, 2 * Kp, Np, BK, true);
    if (rc) return rc;
    TcParams p{};
    p.M = m; p.N = n; p.K = k; p.k_per_split = Kp; p.Kp = Kp;
    p.direct = 1; p.C = C; p.ldc = ldc; p.alpha = alpha; p.beta = beta; p.row_sub = row_sub; p.ws = nullptr;
    p.pred = pred;
    dim3 grid((unsigned)cdiv(m, BM), (unsigned)cdiv(n, bn), 1);
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
    return s * k * n * 4 + 256;
}

int gemm_tn_tc(int out_dtype, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t lda,
               const float* B, int64_t ldb, double beta, void* C, int64_t ldc, const double* mu, const double* cs,
               void* ws, int64_t ws_bytes, const int32_t* pred, cudaStream_t st) {
    // operand view: D[Mop x Nop] = A^T[Mop x Kop] B[Kop x Nop], Mop = k, Kop = m
    const int64_t Mop = k, Nop = n, Kop = m;
    int bn = pick_bn(Nop);
    const int64_t S = tn_splits_tc(Mop, Nop, Kop);
    RSVD_REQUIRE(ws_bytes >= S * Mop * Nop * 4, "gemm_tn_tc: workspace too small");
    const int64_t Kp = cdiv(Kop, BK) * BK, Np = cdiv(Nop, 32) * 32 + 128;
    static thread_local Scratch sc;
    size_t need = (size_t)(2 * Kp * Np * 4);
    if (sc.bytes < need) {
        if (sc.ptr) cudaFreeAsync(sc.ptr, st);
        RSVD_CHECK_CUDA(cudaMallocAsync(&sc.ptr, need, st));
        sc.bytes = need;
    }
    float* bs = (float*)sc.ptr;
    int rc = split_b(B, Kop, Nop, ldb, Kp, Np, bs, pred, st);
    if (rc) return rc;
    CUtensorMap tA, tB;
    rc = make_map(&tA, A, k /*inner = columns of A*/, m, lda, BK, true);
    if (rc) return rc;
    rc = make_map(&tB, bs, Np, 2 * Kp, Np, BK, true);
    if (rc) return rc;
    TcParams p{};
    p.M = Mop; p.N = Nop; p.K = Kop;
    p.k_per_split = cdiv(cdiv(Kop, S), BK) * BK;
    p.Kp = Kp;
    p.direct = 0; p.ws = (float*)ws; p.pred = pred;
    dim3 grid((unsigned)cdiv(Mop, BM), (unsigned)cdiv(Nop, bn), (unsigned)S);
    rc = dispatch_bn<true>(bn, tA, tB, p, grid, st);
    if (rc) return rc;
    int64_t tot = Mop * Nop;
    if (out_dtype == RSVD_F64)
        k_tc_reduce<double><<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(Mop, Nop, S, (const float*)ws, alpha, beta,
                                                                       (double*)C, ldc, mu, cs, pred);
    else
        k_tc_reduce<float><<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(Mop, Nop, S, (const float*)ws, alpha, beta,
                                                                      (float*)C, ldc, mu, cs, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace rsvd
