// Probe: FP64 tensor-core (mma.sync f64, DMMA) throughput vs FP64 FMA on this
// GPU, to size the FP64 parity path. Debug tool, not shipped.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/dmma_probe tools/dmma_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ void dmma_k4(double* c, double a0, double a1, double b0) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a0), "d"(a1), "d"(b0));
}
__device__ __forceinline__ void dmma_k8(double* c, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void dmma_k16(double* c, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                 "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int KIND>
__global__ void thr(double* out, int iters) {
    double c[8][4];
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) c[i][j] = 0;
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
    for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 4) dmma_k4(c[i], a[0], a[1], b[0]);
            if (KIND == 8) dmma_k8(c[i], a, b);
            if (KIND == 16) dmma_k16(c[i], a, b);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) s += c[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma(double* out, int iters, double a) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, 1.0);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 1 << 26);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        int blocks = sms * 2, threads = 32 * warps;
        auto run = [&](auto kern, double flop_per_warp_iter, const char* name) {
            kern<<<blocks, threads>>>(out, iters);
            cudaEventRecord(e0);
            kern<<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fl = flop_per_warp_iter * iters * (double)blocks * warps;
            printf("%-10s warps/blk %2d: %.2f TFLOP/s\n", name, warps, fl / ms / 1e9);
        };
        run(thr<4>, 8.0 * 2 * 16 * 8 * 4, "dmma_k4");
        run(thr<8>, 8.0 * 2 * 16 * 8 * 8, "dmma_k8");
        run(thr<16>, 8.0 * 2 * 16 * 8 * 16, "dmma_k16");
        ffma<<<blocks, threads>>>(out, iters, 0.999);
        cudaEventRecord(e0);
        ffma<<<blocks, threads>>>(out, iters, 0.999);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-10s warps/blk %2d: %.2f TFLOP/s\n", "ffma64", warps,
               2.0 * 8 * 32 * iters * (double)blocks * warps / ms / 1e9);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
