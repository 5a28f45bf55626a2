#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>
#include <random>
__device__ __forceinline__ double warp_sum(double v) { for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o); return v; }
constexpr int kFastP = 224;
constexpr int kFastThreads = 1024;

template <int KR>
__global__ void __launch_bounds__(kFastThreads)
k_chol_fast(int p, const double* __restrict__ G, int64_t ldg, const double* __restrict__ ref2, double tau2,
            double* __restrict__ T, int64_t ldt, int32_t* __restrict__ mask, int32_t* __restrict__ ndef,
            int32_t* __restrict__ running, const int32_t* __restrict__ active, const int32_t* __restrict__ pred, long long* dbg) {
    if (pred && *pred == 0) return;
    extern __shared__ double S[];  // packed upper triangle of the Schur complement / R
    __shared__ double s_ref[kFastP];
    __shared__ double s_rinv[kFastP];  // 1 / R[j][j] (1 for deficient slots)
    __shared__ double s_rdiag[kFastP];
    __shared__ int s_msk[kFastP];
    __shared__ int s_act[kFastP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    auto off = [p](int i, int j) { return i * p - (i * (i - 1)) / 2 + (j - i); };
    for (int i = warp; i < p; i += nwarps)
        for (int j = i + lane; j < p; j += 32) S[off(i, j)] = G[(int64_t)i * ldg + j];
    for (int j = tid; j < p; j += blockDim.x) {
        s_ref[j] = ref2 ? ref2[j] : G[(int64_t)j * ldg + j];
        s_act[j] = active ? active[j] : 1;
    }
    __syncthreads();
    long long t0 = clock64(), tpiv = 0, tupd = 0, tsync = 0;
    int count = 0;
    for (int j = 0; j < p; ++j) {
        long long a0 = clock64();
        // pivot test, redundantly in every thread (factor.py:105 analogue)
        const double d = S[off(j, j)];
        const int act = s_act[j];
        const int def = !act || !(d > tau2 * s_ref[j]) || !(d > 0.0);
        count += def && act;
        long long a1 = clock64(); tpiv += a1 - a0;
        if (!def) {
            const double inv2 = 1.0 / d;
            const double* __restrict__ rj = S + (off(j, j) - j);  // row j, unscaled, read-only this step
            for (int a = j + 1 + warp; a < p; a += nwarps) {
                const double ra = rj[a] * inv2;
                double* __restrict__ rowa = S + (off(a, a) - a);
#pragma unroll 4
                for (int b = a + lane; b < p; b += 32) rowa[b] = fma(-ra, rj[b], rowa[b]);
            }
        }
        if (tid == 0) {
            s_msk[j] = def ? (act ? 1 : 2) : 0;
            const double rjj = def ? 1.0 : sqrt(d);
            s_rdiag[j] = rjj;
            s_rinv[j] = 1.0 / rjj;
        }
        long long a2 = clock64(); tupd += a2 - a1;
        __syncthreads();
        tsync += clock64() - a2;
    }
    long long t1 = clock64();
    // scale the rows of R (deficient rows become e_j)
    for (int i = warp; i < p; i += nwarps) {
        const bool di = s_msk[i] != 0;
        const double inv = s_rinv[i];
        for (int j = i + lane; j < p; j += 32) {
            const int o = off(i, j);
            S[o] = (j == i) ? s_rdiag[i] : (di ? 0.0 : S[o] * inv);
        }
    }
    __syncthreads();
    long long t15 = clock64();
    // rows of T = R^{-1}: row c is s with R^T s = e_c (s_a = 0 for a < c)
    for (int c = warp; c < p; c += nwarps) {
        double x[KR];
#pragma unroll
        for (int r = 0; r < KR; ++r) x[r] = (lane + 32 * r == c) ? 1.0 : 0.0;
        for (int b = c; b < p; ++b) {
            const int rb = b >> 5, lb = b & 31;
            const double* rowb = S + (off(b, b) - b);
            double rrow[KR];
#pragma unroll
            for (int r = 0; r < KR; ++r) {
                const int a = lane + 32 * r;
                rrow[r] = (a > b && a < p) ? rowb[a] : 0.0;
            }
            double xb = 0.0;
#pragma unroll
            for (int r = 0; r < KR; ++r)
                if (r == rb) xb = x[r];
            xb = __shfl_sync(0xffffffffu, xb, lb) * s_rinv[b];
#pragma unroll
            for (int r = 0; r < KR; ++r) {
                const int a = lane + 32 * r;
                x[r] = (a == b) ? xb : fma(-rrow[r], xb, x[r]);
            }
        }
        const bool zc = s_msk[c] != 0;
#pragma unroll
        for (int r = 0; r < KR; ++r) {
            const int a = lane + 32 * r;
            if (a < p) T[(int64_t)c * ldt + a] = (zc || s_msk[a] || a < c) ? 0.0 : x[r];
        }
    }
    __syncthreads();
    long long t2 = clock64();
    if (tid == 0) { dbg[0] = t1 - t0; dbg[1] = t2 - t15; dbg[2] = tpiv; dbg[3] = tupd; dbg[4] = tsync; dbg[5] = t15 - t1; }
    for (int j = tid; j < p; j += blockDim.x) mask[j] = s_msk[j] == 1 ? 1 : 0;
    if (tid == 0) {
        const int32_t base = running ? running[0] : 0;
        ndef[0] = count;
        ndef[1] = base;
        if (running) running[0] = base + count;
    }
}

int main() {
  for (int p : {50, 200}) {
    std::mt19937 g(1); std::normal_distribution<double> nd;
    int n = 2000; std::vector<double> v(n * p), G(p * p, 0.0);
    for (auto& x : v) x = nd(g);
    for (int i = 0; i < p; ++i) for (int j = 0; j < p; ++j) { double s = 0; for (int r = 0; r < n; ++r) s += v[r * p + i] * v[r * p + j]; G[i * p + j] = s; }
    double *dG, *dT; int32_t *dm, *dn; long long* dd;
    cudaMalloc(&dG, p * p * 8); cudaMalloc(&dT, p * p * 8); cudaMalloc(&dm, p * 4); cudaMalloc(&dn, 8); cudaMalloc(&dd, 64);
    cudaMemcpy(dG, G.data(), p * p * 8, cudaMemcpyHostToDevice);
    size_t sm = p * (p + 1) / 2 * 8;
    int threads = 1024;
    cudaFuncSetAttribute(k_chol_fast<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_chol_fast<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int it = 0; it < 3; ++it) {
      if (p <= 64) k_chol_fast<2><<<1, threads, sm>>>(p, dG, p, nullptr, 1e-14, dT, p, dm, dn, nullptr, nullptr, nullptr, dd);
      else k_chol_fast<7><<<1, threads, sm>>>(p, dG, p, nullptr, 1e-14, dT, p, dm, dn, nullptr, nullptr, nullptr, dd);
    }
    cudaError_t e = cudaDeviceSynchronize();
    long long h[6]; cudaMemcpy(h, dd, 48, cudaMemcpyDeviceToHost);
    printf("p=%d err=%s chol=%lld inv=%lld piv=%lld upd=%lld sync=%lld scale=%lld cycles\n", p, cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[5]);
  }
}
