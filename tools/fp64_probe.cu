// Probe: FP64 FMA throughput / latency and division / sqrt cost on this GPU.
// Debug tool, not shipped.
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void thr(double* out, int iters, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, 1.0); x1 = fma(x1, a, 1.0); x2 = fma(x2, a, 1.0); x3 = fma(x3, a, 1.0);
        x4 = fma(x4, a, 1.0); x5 = fma(x5, a, 1.0); x6 = fma(x6, a, 1.0); x7 = fma(x7, a, 1.0);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void thr32(float* out, int iters, float a) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fmaf(x0, a, 1.f); x1 = fmaf(x1, a, 1.f); x2 = fmaf(x2, a, 1.f); x3 = fmaf(x3, a, 1.f);
        x4 = fmaf(x4, a, 1.f); x5 = fmaf(x5, a, 1.f); x6 = fmaf(x6, a, 1.f); x7 = fmaf(x7, a, 1.f);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void lat(double* out, long long* cyc, int iters, double a) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, a, 1.0);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void divlat(double* out, long long* cyc, int iters, double a) {
    double x = threadIdx.x + 2.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = 1.0 / x + a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void sqrtlat(double* out, long long* cyc, int iters, double a) {
    double x = threadIdx.x + 2.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = sqrt(x) + a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void syncl(long long* cyc, int iters) {
    __shared__ volatile int v;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { if (threadIdx.x == 0) v = i; __syncthreads(); }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; float* o32; long long* c;
    cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&o32, 148 * 1024 * 4); cudaMalloc(&c, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int it = 20000;
    thr<<<148 * 4, 256>>>(o, 10, 0.999);
    cudaEventRecord(e0); thr<<<148 * 4, 256>>>(o, it, 0.999); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("FP64 FMA throughput: %.1f TFLOP/s\n", 2.0 * 8 * it * 148.0 * 4 * 256 / ms / 1e9);
    cudaEventRecord(e0); thr32<<<148 * 4, 256>>>(o32, it, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FP32 FMA throughput: %.1f TFLOP/s\n", 2.0 * 8 * it * 148.0 * 4 * 256 / ms / 1e9);
    long long cy;
    lat<<<1, 32>>>(o, c, 10000, 0.999); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", cy / 10000.0);
    divlat<<<1, 32>>>(o, c, 1000, 0.5); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("double 1/x + a dependent: %.1f cycles\n", cy / 1000.0);
    sqrtlat<<<1, 32>>>(o, c, 1000, 0.5); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("double sqrt(x) + a dependent: %.1f cycles\n", cy / 1000.0);
    for (int nt = 64; nt <= 1024; nt *= 4) {
        syncl<<<1, nt>>>(c, 1000); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("__syncthreads (%d threads): %.1f cycles\n", nt, cy / 1000.0);
    }
    return 0;
}
