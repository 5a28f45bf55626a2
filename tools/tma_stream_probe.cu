// Probe: raw TMA streaming bandwidth for the chain-product load pattern
// (A row-major n x d FP32, one CTA per 128-row tile, boxes of 128 rows x 32
// k-elements = 128 B per row, SWIZZLE_128B). No MMA: one consumer warp waits
// on full[s] and immediately frees the stage. Varies boxes-per-stage (bytes
// per row per request) and pipeline depth. Debug tool, not shipped.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(b)), "r"(ph));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
                 "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
                 : "memory");
}

constexpr int BOX_BYTES = 128 * 128;

__global__ void __launch_bounds__(64) k_stream(const __grid_constant__ CUtensorMap tm, int kblocks, int ntiles,
                                              int stages, int boxes, float* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[16], empty[16];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int steps = kblocks / boxes;
    if (warp == 0 && lane == 0) {
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int kb = 0; kb < steps; ++kb, ++it) {
                const int s = it % stages;
                if (it >= stages) mbar_wait(&empty[s], ((it / stages) - 1) & 1);
                mbar_expect(&full[s], boxes * BOX_BYTES);
                for (int b = 0; b < boxes; ++b)
                    tma2d(smem + (size_t)(s * boxes + b) * BOX_BYTES, &tm, &full[s], (kb * boxes + b) * 32, tile * 128);
            }
    } else if (warp == 1) {
        int it = 0;
        float acc = 0.f;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int kb = 0; kb < steps; ++kb, ++it) {
                const int s = it % stages;
                mbar_wait(&full[s], (it / stages) & 1);
                acc += *(volatile float*)(smem + (size_t)s * boxes * BOX_BYTES + lane * 4);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        if (acc == 12345.f) sink[0] = acc;
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int64_t n = 50048, d = 10016;  // multiples of 128 / 32
    float* A;
    cudaMalloc(&A, n * d * 4);
    cudaMemset(A, 0, n * d * 4);
    float* sink;
    cudaMalloc(&sink, 4);
    void* fp;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fp;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int promo = 0; promo < 2; ++promo) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
        cuuint64_t strides[1] = {(cuuint64_t)d * 4};
        cuuint32_t box[2] = {32, 128};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int ntiles = (int)(n / 128), kblocks = (int)(d / 32);
        int cfgs[][3] = {{1, 4, 0}, {1, 6, 0}, {1, 8, 0}, {1, 12, 0}, {2, 3, 0}, {2, 6, 0}, {4, 3, 0},
                         {1, 6, 1}, {2, 3, 1}, {1, 4, 2}, {1, 6, 3}};
        for (auto& c : cfgs) {
            const int boxes = c[0], stages = c[1], grid_mode = c[2];
            const size_t sm = (size_t)boxes * stages * BOX_BYTES + 1024;
            cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            // grid_mode 0: one CTA per tile; 1: persistent (sms); 2: 2 per SM persistent (small smem); 3: 3x sms
            int grid = grid_mode == 0 ? ntiles : grid_mode == 1 ? sms : grid_mode == 2 ? 2 * sms : 3 * sms;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int w = 0; w < 2; ++w) k_stream<<<grid, 64, sm>>>(tm, kblocks, ntiles, stages, boxes, sink);
            cudaEventRecord(e0);
            const int R = 5;
            for (int r = 0; r < R; ++r) k_stream<<<grid, 64, sm>>>(tm, kblocks, ntiles, stages, boxes, sink);
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= R;
            printf("promo %d boxes %d stages %2d grid %5d (%d): %.3f ms  %.0f GB/s  %s\n", promo, boxes, stages, grid,
                   grid_mode, ms, n * d * 4 / ms / 1e6, cudaGetErrorString(e));
        }
    }
    return 0;
}
