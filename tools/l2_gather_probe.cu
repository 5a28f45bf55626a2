// Probe: the L2 -> SM row-gather ceiling that bounds the CSR products (C3).
// A table of R rows x NB floats (L2-resident, 40 MB at R = 1e5, NB = 100)
// is gathered by N random row indices (uniform over the rows); each gathered
// row is summed into per-lane accumulators, so the work per row is what a
// CSR product does per nonzero minus the value multiply.
//   ldg  : warp per 32 indices, U rows in flight per warp, float4 lanes
//   bulk : warp per 32 indices, each warp a private smem ring of S row slots
//          filled by cp.async.bulk (lane 0), mbarrier per slot, LDS.128 reads
// Reports gathered GB/s (N x row bytes / time). Debug tool, not shipped.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/l2_gather_probe tools/l2_gather_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int U>
__global__ void __launch_bounds__(256) k_ldg(const float* __restrict__ T, int ld, int nb, const int* __restrict__ idx,
                                             int64_t n, float* sink) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool on = 4 * lane < nb;
    for (int64_t base = w * 32; base < n; base += nw * 32) {
        const int my = base + lane < n ? idx[base + lane] : 0;
        const int cnt = (int)min((int64_t)32, n - base);
        int i = 0;
        for (; i + U <= cnt; i += U) {
            int r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = __shfl_sync(0xffffffffu, my, i + u);
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                v[u] = on ? *reinterpret_cast<const float4*>(T + (int64_t)r[u] * ld + 4 * lane) : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
            }
        }
        for (; i < cnt; ++i) {
            const int r = __shfl_sync(0xffffffffu, my, i);
            if (on) {
                float4 v = *reinterpret_cast<const float4*>(T + (int64_t)r * ld + 4 * lane);
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) sink[0] = 1.f;
}

// like k_ldg<8> but shaped like k_spmm_nnz_f32: each warp owns a contiguous run of
// RUN indices, multiplies by a per-index value and shuffles a row id along
template <int U, int RUN>
__global__ void __launch_bounds__(256, 3) k_run(const float* __restrict__ T, int ld, int nb, const int* __restrict__ idx,
                                                const float* __restrict__ val, int64_t n, float* sink) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool on = 4 * lane < nb;
    const int64_t nruns = (n + RUN - 1) / RUN;
    for (int64_t run = w; run < nruns; run += nw) {
        const int64_t e0 = run * RUN, e1 = min(n, e0 + RUN);
        for (int64_t base = e0; base < e1; base += 32) {
            const int my = base + lane < e1 ? idx[base + lane] : 0;
            const float mv = base + lane < e1 ? val[base + lane] : 0.f;
            const int cnt = (int)min((int64_t)32, e1 - base);
            for (int i = 0; i < cnt; i += U) {
                int r[U];
                float vv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    r[u] = __shfl_sync(0xffffffffu, my, i + u);
                    vv[u] = __shfl_sync(0xffffffffu, mv, i + u);
                }
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    v[u] = on ? *reinterpret_cast<const float4*>(T + (int64_t)r[u] * ld + 4 * lane) : make_float4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    acc.x = fmaf(vv[u], v[u].x, acc.x); acc.y = fmaf(vv[u], v[u].y, acc.y);
                    acc.z = fmaf(vv[u], v[u].z, acc.z); acc.w = fmaf(vv[u], v[u].w, acc.w);
                }
            }
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) sink[0] = 1.f;
}

// k_run + row ids: a finished row is flushed (MODE 1: the flush only counts; MODE 2: it stores the row)
template <int U, int RUN, int MODE>
__global__ void __launch_bounds__(256, 3) k_rows(const float* __restrict__ T, int ld, int nb, const int* __restrict__ idx,
                                                 const float* __restrict__ val, const int* __restrict__ rowid, int64_t n,
                                                 float* __restrict__ C, float* sink) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool on = 4 * lane < nb;
    const int64_t nruns = (n + RUN - 1) / RUN;
    float tot = 0.f;
    for (int64_t run = w; run < nruns; run += nw) {
        const int64_t e0 = run * RUN, e1 = min(n, e0 + RUN);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        int cur = -1;
        for (int64_t base = e0; base < e1; base += 32) {
            const bool in = base + lane < e1;
            const int my = in ? idx[base + lane] : 0;
            const float mv = in ? val[base + lane] : 0.f;
            int rr = in ? rowid[base + lane] : 0;
            const int cnt = (int)min((int64_t)32, e1 - base);
            const int rl = __shfl_sync(0xffffffffu, rr, cnt - 1);
            rr = lane < cnt ? rr : rl;
            for (int i = 0; i < cnt; i += U) {
                int r[U], ro[U];
                float vv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    r[u] = __shfl_sync(0xffffffffu, my, i + u);
                    vv[u] = __shfl_sync(0xffffffffu, mv, i + u);
                    ro[u] = __shfl_sync(0xffffffffu, rr, i + u);
                }
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    v[u] = on ? *reinterpret_cast<const float4*>(T + (int64_t)r[u] * ld + 4 * lane) : make_float4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (ro[u] != cur) {
                        if (cur >= 0) {
                            if (MODE == 2) {
                                if (on) *reinterpret_cast<float4*>(C + (int64_t)cur * ld + 4 * lane) = acc;
                            } else {
                                tot += acc.x + acc.y + acc.z + acc.w;
                            }
                        }
                        cur = ro[u];
                        acc = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    acc.x = fmaf(vv[u], v[u].x, acc.x); acc.y = fmaf(vv[u], v[u].y, acc.y);
                    acc.z = fmaf(vv[u], v[u].z, acc.z); acc.w = fmaf(vv[u], v[u].w, acc.w);
                }
            }
        }
        if (cur >= 0) {
            if (MODE == 2) {
                if (on) *reinterpret_cast<float4*>(C + (int64_t)cur * ld + 4 * lane) = acc;
            } else {
                tot += acc.x + acc.y + acc.z + acc.w;
            }
        }
    }
    if (tot == 1234.5f) sink[0] = 1.f;
}

template <int S>
__global__ void __launch_bounds__(256) k_bulk(const float* __restrict__ T, int ld, int nb, const int* __restrict__ idx,
                                              int64_t n, float* sink) {
    extern __shared__ __align__(16) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[8][S];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int rowb = nb * 4;
    float* ring = reinterpret_cast<float*>(sm + (size_t)wid * S * rowb);
    if (lane < S) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[wid][lane])));
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool on = 4 * lane < nb;
    uint32_t phase[S];
#pragma unroll
    for (int s = 0; s < S; ++s) phase[s] = 0;
    for (int64_t base = w * 32; base < n; base += nw * 32) {
        const int my = base + lane < n ? idx[base + lane] : 0;
        const int cnt = (int)min((int64_t)32, n - base);
        // prologue: S copies in flight
        auto issue = [&](int i) {
            const int r = __shfl_sync(0xffffffffu, my, i);
            const int s = i % S;
            if (lane == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[wid][s])),
                             "r"(rowb));
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(ring + s * nb)),
                    "l"(T + (int64_t)r * ld), "r"(rowb), "r"(smem_u32(&bar[wid][s]))
                    : "memory");
            }
        };
        for (int i = 0; i < S && i < cnt; ++i) issue(i);
        for (int i = 0; i < cnt; ++i) {
            const int s = i % S;
            uint32_t ph = 0;
#pragma unroll
            for (int q = 0; q < S; ++q)
                if (q == s) ph = phase[q];
            asm volatile(
                "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra "
                "D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar[wid][s])),
                "r"(ph));
#pragma unroll
            for (int q = 0; q < S; ++q)
                if (q == s) phase[q] ^= 1u;
            if (on) {
                float4 v = *reinterpret_cast<const float4*>(ring + s * nb + 4 * lane);
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
            __syncwarp();
            if (i + S < cnt) issue(i + S);
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) sink[0] = 1.f;
}

int main(int argc, char** argv) {
    const int R = 100000, nb = 100, ld = argc > 1 ? atoi(argv[1]) : 100;
    const int64_t n = 10000000;
    float *T, *sink;
    int* idx;
    cudaMalloc(&T, (size_t)R * ld * 4);
    cudaMalloc(&sink, 4);
    cudaMalloc(&idx, n * 4);
    cudaMemset(T, 0, (size_t)R * ld * 4);
    int* h = (int*)malloc(n * 4);
    uint64_t s = 88172645463325252ull;
    for (int64_t i = 0; i < n; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        h[i] = (int)(s % R);
    }
    cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = (double)n * nb * 4;
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        printf("%-28s ld %3d  %.3f ms  %.0f GB/s gathered\n", name, ld, ms, bytes / ms / 1e6);
        cudaError_t err = cudaGetLastError();
        if (err) printf("  error %s\n", cudaGetErrorString(err));
    };
    for (int ctas : {2, 3, 4, 8}) {
        char nm[64];
        snprintf(nm, 64, "ldg U=2 ctas/sm=%d", ctas);
        run(nm, [&] { k_ldg<2><<<sms * ctas, 256>>>(T, ld, nb, idx, n, sink); });
        snprintf(nm, 64, "ldg U=4 ctas/sm=%d", ctas);
        run(nm, [&] { k_ldg<4><<<sms * ctas, 256>>>(T, ld, nb, idx, n, sink); });
        snprintf(nm, 64, "ldg U=8 ctas/sm=%d", ctas);
        run(nm, [&] { k_ldg<8><<<sms * ctas, 256>>>(T, ld, nb, idx, n, sink); });
    }
    {
        float* val;
        cudaMalloc(&val, n * 4);
        cudaMemset(val, 0, n * 4);
        for (int ctas : {3, 4}) {
            char nm[64];
            snprintf(nm, 64, "run1024 U=8 ctas/sm=%d", ctas);
            run(nm, [&] { k_run<8, 1024><<<sms * ctas, 256>>>(T, ld, nb, idx, val, n, sink); });
            snprintf(nm, 64, "run32 U=8 ctas/sm=%d", ctas);
            run(nm, [&] { k_run<8, 32><<<sms * ctas, 256>>>(T, ld, nb, idx, val, n, sink); });
        }
        int* rowid;
        float* C;
        cudaMalloc(&rowid, n * 4);
        cudaMalloc(&C, (size_t)200000 * ld * 4);
        int* hr = (int*)malloc(n * 4);
        for (int64_t i = 0; i < n; ++i) hr[i] = (int)(i / 54);
        cudaMemcpy(rowid, hr, n * 4, cudaMemcpyHostToDevice);
        run("rows54 count U=8 ctas/sm=3", [&] { k_rows<8, 1024, 1><<<sms * 3, 256>>>(T, ld, nb, idx, val, rowid, n, C, sink); });
        run("rows54 store U=8 ctas/sm=3", [&] { k_rows<8, 1024, 2><<<sms * 3, 256>>>(T, ld, nb, idx, val, rowid, n, C, sink); });
        // lognormal-ish row lengths: alternate short (5) and long (103) rows, mean 54
        { int64_t e = 0; int row = 0; while (e < n) { int len = (row & 1) ? 103 : 5; for (int k = 0; k < len && e < n; ++k) hr[e++] = row; ++row; } }
        cudaMemcpy(rowid, hr, n * 4, cudaMemcpyHostToDevice);
        run("rows5/103 store U=8 ctas/sm=3", [&] { k_rows<8, 1024, 2><<<sms * 3, 256>>>(T, ld, nb, idx, val, rowid, n, C, sink); });
    }
    if (argc > 2) return 0;
    {
        const int smb4 = 8 * 4 * nb * 4, smb8 = 8 * 8 * nb * 4, smb16 = 8 * 16 * nb * 4;
        cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb4);
        cudaFuncSetAttribute(k_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb8);
        cudaFuncSetAttribute(k_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb16);
        for (int ctas : {2, 4, 8}) {
            char nm[64];
            snprintf(nm, 64, "bulk S=4 ctas/sm=%d", ctas);
            run(nm, [&] { k_bulk<4><<<sms * ctas, 256, smb4>>>(T, ld, nb, idx, n, sink); });
            snprintf(nm, 64, "bulk S=8 ctas/sm=%d", ctas);
            run(nm, [&] { k_bulk<8><<<sms * ctas, 256, smb8>>>(T, ld, nb, idx, n, sink); });
            if (ctas <= 2) {
                snprintf(nm, 64, "bulk S=16 ctas/sm=%d", ctas);
                run(nm, [&] { k_bulk<16><<<sms * ctas, 256, smb16>>>(T, ld, nb, idx, n, sink); });
            }
        }
    }
    return 0;
}
