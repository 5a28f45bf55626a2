// Probe: issue cost of tcgen05.mma.kind::tf32 shapes used by the chain GEMM,
// with operands resident in smem / TMEM (no TMA), optionally with 4 warps
// streaming LDS.128 over a 16 KB smem tile (the converters' read traffic).
// One CTA per SM; cycles per k-step (K=8) measured on the MMA thread.
// Debug tool, not shipped.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amn, int bmn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}

// mode: 0 SS N=64; 1 SS N=128; 2 TS N=64; 3 TS N=128; 4 SS N=128 + TS N=64 (current kernel);
//       5 TS N=128 + TS N=64 (A_hi and A_lo both in TMEM); 6 SS N=64 x3 (old kernel, K-major B);
//       7 SS N=256; 8 TS N=256. ROT = accumulators rotated over consecutive k-steps.
template <int MODE, int ROT, int CE, int NC>
__global__ void __launch_bounds__(128, 1) k_probe(int ksteps, long long* out, int rnd, int sttm) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t cbar[4];
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + 12345u;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        ((float*)smem)[i] = rnd ? ((float)(h & 0xFFFFFF) / 16777216.f - 0.5f) : 0.f;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cbar[i])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tslot;
    {   // A operand columns 384..511 of TMEM: random or zero, every lane quarter
        uint32_t v[16];
        for (int c = 384; c < 512; c += 16) {
            for (int j = 0; j < 16; ++j) {
                uint32_t h = (uint32_t)(threadIdx.x * 977 + c * 31 + j) * 2654435761u;
                h ^= h >> 15;
                v[j] = __float_as_uint(rnd ? ((float)(h & 0xFFFFFF) / 16777216.f - 0.5f) : 0.f);
            }
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tb + ((uint32_t)(warp * 32) << 16) + c),
                         "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    constexpr int NW = (MODE == 1 || MODE == 3 || MODE == 4 || MODE == 5) ? 128 : (MODE >= 7 ? 256 : 64);
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
        const uint64_t da0 = make_desc(a, 16, 1024, 2), db0 = make_desc(b, 16, 1024, 2);
        long long t0 = clock64();
        constexpr int UN = (CE > 4 * ROT) ? CE : 4 * ROT;
        for (int it = 0; it < ksteps; it += UN) {
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                const int ks = u & 3;
                const uint64_t da = da0 + 2 * ks, db = db0 + 2 * ks;
                const uint32_t ta = tb + 384 + ks * 8, ta2 = tb + 448 + ks * 8;
                const uint32_t d = tb + (u % ROT) * (MODE == 6 ? 128 : NW);
                switch (MODE) {
                    case 0: mma_ss(d, da, db, idesc(128, 64, 0, 0), 1); break;
                    case 1: mma_ss(d, da, db, idesc(128, 128, 0, 0), 1); break;
                    case 2: mma_ts(d, ta, db, idesc(128, 64, 0, 0), 1); break;
                    case 3: mma_ts(d, ta, db, idesc(128, 128, 0, 0), 1); break;
                    case 4: mma_ss(d, da, db, idesc(128, 128, 0, 0), 1); mma_ts(d, ta2, db, idesc(128, 64, 0, 0), 1); break;
                    case 5: mma_ts(d, ta, db, idesc(128, 128, 0, 0), 1); mma_ts(d, ta2, db, idesc(128, 64, 0, 0), 1); break;
                    case 6:
                        mma_ss(d, da, db, idesc(128, 64, 0, 0), 1);
                        mma_ss(d + 64, da, db, idesc(128, 64, 0, 0), 1);
                        mma_ss(d, da, db, idesc(128, 64, 0, 0), 1);
                        break;
                    case 7: mma_ss(d, da, db, idesc(128, 256, 0, 0), 1); break;
                    case 8: mma_ts(d, ta, db, idesc(128, 256, 0, 0), 1); break;
                }
                if (CE && ((u + 1) % (CE ? CE : 1)) == 0)
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&cbar[c])));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)), "r"(0));
        long long t1 = clock64();
        done = 1;
        if (blockIdx.x == 0) out[0] = t1 - t0;
    } else if (sttm && warp >= 1) {
        // converter-like TMEM store traffic into columns 320..383 (unused by the MMAs)
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) v[j] = __float_as_uint((float)(j + threadIdx.x));
        while (!done) {
            for (int c = 320; c < 384; c += 16)
                asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tb + ((uint32_t)(warp * 32) << 16) + c),
                             "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
            asm volatile("tcgen05.wait::st.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int MODE, int ROT, int CE = 0, int NC = 0>
void run(const char* name, long long* out, int rnd = 0, int sttm = 0) {
    const int ce = CE, nc = NC;
    const int sm = 64 * 1024 + 1024, ks = 48000;
    cudaFuncSetAttribute(k_probe<MODE, ROT, CE, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    k_probe<MODE, ROT, CE, NC><<<148, 128, sm>>>(ks, out, rnd, sttm);
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc;
    cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("commit every %d x%d | rnd %d sttm %d rot %d  %-18s : %6.1f cyc / k-step  %s\n", ce, nc, rnd, sttm, ROT, name, (double)cyc / ks, cudaGetErrorString(e));
}


template <int FEAT>
__global__ void __launch_bounds__(384, 1) k_kernel_like(int nkb, long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bars[8];
    __shared__ volatile int done_flag;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) done_flag = 0;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + 12345u;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        ((float*)smem)[i] = (float)(h & 0xFFFFFF) / 16777216.f - 0.5f;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[i])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tslot;
    const int lane = threadIdx.x % 32;
    if ((FEAT & 8) ? (warp == 0) : (threadIdx.x == 0)) {
        const uint32_t b0 = smem_u32(smem + ((FEAT & 16) ? 131072 : 16384));
        constexpr uint32_t id2 = idesc(128, 128, 0, 0), id1 = idesc(128, 64, 0, 0);
        long long t0 = clock64();
        int chunk = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            const int set = (FEAT & 1) ? (chunk & 1) : 0;
            const uint32_t d0 = tb + set * 128;
            const int st = (FEAT & 2) ? (kb & 3) : 0;
            const uint32_t ta = tb + 256 + st * 64;
            if (FEAT & 64) {
                // satisfied wait (parity 1 of a barrier still in phase 0) + tcgen05 fence
                asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bars[5])), "r"(1), "r"(0x989680));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            if ((FEAT & 32) && lane == 0) out[8 + (kb & 511)] = clock64();
            if (lane == 0) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t db = make_desc(b0 + ks * 32, 16, 1024, 2);
                const uint32_t acc = ((FEAT & 1) ? (kb % 4 > 0 || ks > 0) : 1) ? 1u : 0u;
                mma_ts(d0, ta + ks * 8, db, id2, acc);
                mma_ts(d0, ta + 32 + ks * 8, db, id1, 1u);
            }
            if (FEAT & 32) out[1024 + (kb & 511)] = clock64();
            if (FEAT & 4) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[0])));
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[1])));
                if (kb % 4 == 3) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[2])));
            }
            }
            if (FEAT & 8) __syncwarp();
            if (kb % 4 == 3) ++chunk;
        }
        if (lane == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[7])));
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bars[7])), "r"(0));
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
        }
        if (FEAT & 8) __syncwarp();
        if (threadIdx.x == 0) done_flag = 1;
    } else if ((FEAT & 128) && warp >= 2) {
        // busy neighbours: ALU + LDS loops until the MMA thread finishes
        float acc = 0.f;
        const float* sp = (const float*)smem;
        int i = threadIdx.x;
        while (!done_flag) {
#pragma unroll 16
            for (int j = 0; j < 16; ++j) acc = fmaf(acc, 1.0001f, sp[(i + j * 33) & 16383]);
            i += 7;
        }
        if (acc == 1.f) out[2000] = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int FEAT>
void run_kl(long long* out) {
    const int sm = 192 * 1024 + 1024, nkb = 12000;
    cudaFuncSetAttribute(k_kernel_like<FEAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    k_kernel_like<FEAT><<<148, 384, sm>>>(nkb, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc;
    cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("kernel-like feat %d (chunk-switch %d, A-stage-rot %d, commits %d): %7.1f cyc / k-block  %s\n", FEAT,
           FEAT & 1, (FEAT >> 1) & 1, (FEAT >> 2) & 1, (double)cyc / nkb, cudaGetErrorString(e));
}

int main() {
    long long* out;
    cudaMalloc(&out, 8 * 2048);
    run<5, 1, 0, 0>("TS N128 + TS N64", out, 1);
    run_kl<7>(out); run_kl<71>(out); run_kl<135>(out); run_kl<199>(out);
    return 0;
}
