// Standalone probe of the tcgen05 building blocks used by gemm_tc.cu
// (TMEM alloc/st/ld round trip; one kind::tf32 MMA from hand-written
// SWIZZLE_128B smem tiles, K-major and MN-major). Debug tool, not shipped.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
// 128B rows, 32-byte chunks swizzled with (row % 4)  (Swizzle<2,5,2>)
__device__ __forceinline__ int sw128_32(int r, int c) {
    int chunk = c / 8, within = c % 8;
    return r * 128 + ((chunk ^ (r % 4)) * 32) + within * 4;
}

__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int amn, int bmn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// byte offset of element (r, c) (r = row of a 128B-row tile, c = fp32 index in row)
__device__ __forceinline__ int sw128(int r, int c) {
    int chunk = c / 4, within = c % 4;
    return r * 128 + ((chunk ^ (r % 8)) * 16) + within * 4;
}

__global__ void probe(float* out, int mode, int var) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tb = tslot;
    if (threadIdx.x == 0) out[1000] = (float)tb;
    const int quarter = warp % 4;
    const uint32_t laddr = tb + ((uint32_t)(quarter * 32) << 16);
    if (mode == 0) {
        // TMEM st/ld round trip
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) v[i] = __float_as_uint((float)(threadIdx.x * 10 + i));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(laddr), "r"(v[0]),
                     "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(laddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int i = 0; i < 8; ++i) out[threadIdx.x * 8 + i] = __uint_as_float(r[i]);
    } else {
        // A: 128 x 32 (M x K), B: 32 x 32 (K x N). A[m][k] = (m % 7) + k * 0.5, B[k][n] = (k == n) ? 1 : 0
        float* a = (float*)smem;
        float* b = (float*)(smem + 16384);
        const bool a_mn = (mode == 2);
        for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
            int m = e / 32, k = e % 32;
            float val = (float)(m % 7) + k * 0.5f;
            if (!a_mn) {
                *(float*)((uint8_t*)a + sw128(m, k)) = val;  // rows = m, 128B rows of K
            } else {
                // MN-major: atoms of 32 M x 32 K-rows: atom (m/32) at 4096*(m/32), row = k
                *(float*)((uint8_t*)a + (m / 32) * 4096 + sw128_32(k, m % 32)) = val;
            }
        }
        for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
            int k = e / 32, n = e % 32;
            *(float*)((uint8_t*)b + sw128_32(k, n)) = (k == n) ? 1.f : 0.f;  // MN-major: rows = k, 128B of N
        }
        if (var & 4) {
            uint32_t v[8];
            for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(100.f);
            for (int c = 0; c < 32; c += 8)
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(laddr + c), "r"(v[0]),
                             "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
            asm volatile("tcgen05.wait::st.sync.aligned;");
        }
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (threadIdx.x == 32) {
            uint32_t idesc = make_idesc(128, 32, a_mn ? 1 : 0, 1);
            if (var & 2) idesc = (idesc & ~(0x1Fu << 24)) | ((128u >> 4) << 23);
            for (int ks = 0; ks < 4; ++ks) {
                uint64_t da = a_mn ? make_desc(smem_u32(a) + ks * 1024, 4096, 512, 1) : make_desc(smem_u32(a) + ks * 32, 16, 1024);
                uint64_t db = make_desc(smem_u32(b) + ks * 1024, 4096, 512, 1);
                uint32_t acc = (ks > 0) || (var & 4);
                if (var & 1) {
                    uint32_t z = 0;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(tb),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(z));
                } else {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        }
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)), "r"(0));
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int c = 0; c < 32; c += 8) {
            uint32_t r[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "r"(laddr + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            int row = quarter * 32 + lane;
            for (int i = 0; i < 8; ++i) out[row * 32 + c + i] = __uint_as_float(r[i]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(64));
}

int main() {
    float* d;
    cudaMalloc(&d, 8192 * 4);
    float h[8192];
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int it = 0; it < 1 + 2 * 8; it += (it == 0 ? 1 : 4)) {
        int mode = it == 0 ? 0 : 1 + (it - 1) / 8;
        int var = it == 0 ? 0 : (it - 1) % 8;
        cudaMemset(d, 0, 8192 * 4);
        probe<<<1, 128, 64 * 1024>>>(d, mode, var);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8192 * 4, cudaMemcpyDeviceToHost);
        printf("mode %d var %d err=%s\n", mode, var, cudaGetErrorString(e));
        if (mode == 0) {
            int bad = 0;
            for (int t = 0; t < 128; ++t)
                for (int i = 0; i < 8; ++i)
                    if (h[t * 8 + i] != (float)(t * 10 + i)) bad++;
            printf("  roundtrip bad=%d sample %g %g %g\n", bad, h[0], h[9], h[127 * 8 + 7]);
        } else {
            int bad = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 32; ++n) {
                    float ref = (float)(m % 7) + n * 0.5f;
                    if (h[m * 32 + n] != ref) bad++;
                }
            printf("  mma bad=%d  D[0][0..3]=%g %g %g %g  D[5][7]=%g (ref %g) D[100][31]=%g\n", bad, h[0], h[1], h[2], h[3],
                   h[5 * 32 + 7], 5 + 3.5, h[100*32+31]);
        }
    }
    return 0;
}
