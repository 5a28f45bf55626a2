// Probe 3: (a) how kind::tf32 consumes raw FP32 operands (truncate / round /
// full precision); (b) the .ts form: A operand from TMEM (lane = row,
// column = k, one 32-bit column per element), B from smem (K-major SW128).
// Debug tool, not shipped.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

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
__device__ __forceinline__ int sw128(int r, int byte_in_row) {
    int chunk = byte_in_row / 16, within = byte_in_row % 16;
    return r * 128 + ((chunk ^ (r % 8)) * 16) + within;
}

// A: 128 x 32 (K-major), B: 64 x 32 (N x K, K-major). D = A B^T (128 x 64).
// mode 0: A via smem desc; mode 1: A via TMEM (.ts form).
__global__ void probe(float* out, const float* A, const float* B, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tslot;  // D at columns [0,64), A (mode 1) at columns [64, 96)
    const int quarter = warp % 4;
    uint8_t* a = smem;
    uint8_t* b = smem + 16384;
    for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
        int m = e / 32, k = e % 32;
        *(float*)(a + sw128(m, k * 4)) = A[m * 32 + k];
    }
    for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
        int n = e / 32, k = e % 32;
        *(float*)(b + sw128(n, k * 4)) = B[n * 32 + k];
    }
    if (mode == 1) {
        // thread (quarter q, lane l) owns row 32q + l: store its 32 A values into TMEM columns 64..95
        const int row = quarter * 32 + lane;
        uint32_t v[32];
        for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(A[row * 32 + k]);
        const uint32_t taddr = tb + ((uint32_t)(quarter * 32) << 16) + 64;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 32) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int ks = 0; ks < 4; ++ks) {
            const uint64_t db = make_desc(smem_u32(b) + ks * 32, 16, 1024, 2);
            const uint32_t acc = ks > 0;
            if (mode == 0) {
                const uint64_t da = make_desc(smem_u32(a) + ks * 32, 16, 1024, 2);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
                             "l"(da), "l"(db), "r"(idesc), "r"(acc));
            } else {
                const uint32_t ta = tb + 64 + ks * 8;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
                             "r"(ta), "l"(db), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)), "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t laddr = tb + ((uint32_t)(quarter * 32) << 16);
    for (int c = 0; c < 64; c += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(laddr + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const int row = quarter * 32 + lane;
        for (int i = 0; i < 8; ++i) out[row * 64 + c + i] = __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(128));
}

int main() {
    static float hA[128 * 32], hB[64 * 32], hD[128 * 64];
    // rounding probe: A[m][0] = 1 + 3*2^-12 (tf32 trunc -> 1, rna -> 1+2^-10), A[m][1] = 1 + 2^-12
    for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 32; ++k) hA[m * 32 + k] = (float)((m % 5) + 1) * 0.25f + (float)k / 64.f;
    hA[0 * 32 + 0] = 1.0f + 3.0f / 4096.f;
    hA[1 * 32 + 0] = 1.0f + 1.0f / 4096.f;
    hA[2 * 32 + 0] = -(1.0f + 3.0f / 4096.f);
    for (int n = 0; n < 64; ++n)
        for (int k = 0; k < 32; ++k) hB[n * 32 + k] = (n == k) ? 1.f : 0.f;  // D[m][n] = A[m][n] for n < 32
    float *dA, *dB, *dD;
    cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, sizeof(hD));
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dD, 0, sizeof(hD));
        probe<<<1, 128, 64 * 1024>>>(dD, dA, dB, mode);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 3; m < 128; ++m)
            for (int n = 0; n < 32; ++n)
                if (hD[m * 64 + n] != hA[m * 32 + n]) bad++;
        printf("mode %d (%s) err=%s bad(rows>=3, exact tf32 values)=%d\n", mode, mode ? "A in TMEM" : "A in smem",
               cudaGetErrorString(e), bad);
        printf("  1+3*2^-12 -> %.9f  (trunc 1.0, rna %.9f, fp32 %.9f)\n", hD[0], 1.0 + 1.0 / 1024, 1.0 + 3.0 / 4096);
        printf("  1+1*2^-12 -> %.9f ; -(1+3*2^-12) -> %.9f\n", hD[64], hD[128]);
    }
    return 0;
}
