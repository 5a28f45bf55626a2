// Probe 2: one CTA, both operands K-major SWIZZLE_128B, single K=one 128B row.
// mode 0: kind::f16 bf16 (K=64 per row, 4 MMAs of K=16); mode 1: kind::tf32
// (K=32 per row, 4 MMAs of K=8). D = A B^T with A[m][k] = (m%7)+k/8, B[n][k] = (n==k).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int version, int layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)version << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

__device__ __forceinline__ int sw128(int r, int byte_in_row) {
    int chunk = byte_in_row / 16, within = byte_in_row % 16;
    return r * 128 + ((chunk ^ (r % 8)) * 16) + within;
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
    const uint32_t tb = tslot;
    const int quarter = warp % 4;
    const uint32_t laddr = tb + ((uint32_t)(quarter * 32) << 16);
    uint8_t* a = smem;           // 128 rows x 128 B
    uint8_t* b = smem + 16384;   // 64 rows x 128 B (N = 64)
    const int N = 64;
    const int esz = mode == 0 ? 2 : 4;
    const int kdim = 128 / esz;  // elements per row
    for (int e = threadIdx.x; e < 128 * kdim; e += blockDim.x) {
        int m = e / kdim, k = e % kdim;
        float v = (float)(m % 7) + k * 0.125f;
        if (mode == 0) *(__nv_bfloat16*)(a + sw128(m, k * 2)) = __float2bfloat16(v);
        else *(float*)(a + sw128(m, k * 4)) = v;
    }
    for (int e = threadIdx.x; e < N * kdim; e += blockDim.x) {
        int n = e / kdim, k = e % kdim;
        float v = (n == k) ? 1.f : 0.f;
        if (mode == 0) *(__nv_bfloat16*)(b + sw128(n, k * 2)) = __float2bfloat16(v);
        else *(float*)(b + sw128(n, k * 4)) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 32) {
        // idesc: c F32, a/b format, K-major both, N, M
        uint32_t fmt = mode == 0 ? 1u : 2u;  // BF16 / TF32
        uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        int version = (var & 1) ? 0 : 1;
        uint32_t lbo = (var & 2) ? 0 : 16;
        for (int ks = 0; ks < 4; ++ks) {
            uint64_t da = make_desc(smem_u32(a) + ks * 32, lbo, 1024, version, 2);
            uint64_t db = make_desc(smem_u32(b) + ks * 32, lbo, 1024, version, 2);
            uint32_t acc = ks > 0;
            if (mode == 0)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
                             "l"(da), "l"(db), "r"(idesc), "r"(acc));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
                             "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)), "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < N; c += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(laddr + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        int row = quarter * 32 + lane;
        for (int i = 0; i < 8; ++i) out[row * N + c + i] = __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(64));
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 64 * 4);
    static float h[128 * 64];
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int mode = 0; mode < 2; ++mode)
        for (int var = 0; var < 4; ++var) {
            cudaMemset(d, 0, sizeof(h));
            probe<<<1, 128, 64 * 1024>>>(d, mode, var);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            int kdim = mode == 0 ? 64 : 32;
            int bad = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 64; ++n) {
                    float ref = n < kdim ? (float)(m % 7) + n * 0.125f : 0.f;
                    if (fabsf(h[m * 64 + n] - ref) > 1e-2f) bad++;
                }
            printf("mode %d var %d err=%s bad=%d D[5][7]=%g D[3][1]=%g\n", mode, var, cudaGetErrorString(e), bad,
                   h[5 * 64 + 7], h[3 * 64 + 1]);
        }
    return 0;
}
