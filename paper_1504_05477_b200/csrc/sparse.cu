// CSR products: spmm_nt (_kernels.pyx:74-92) and, on the CSR of A^T built
// once per operator, spmm_t (_kernels.pyx:95-113) as a deterministic gather
// (no atomics). Warp per row: the warp loads 32 (col, val) pairs at a time,
// broadcasts each with a shuffle, and every lane accumulates NPL contiguous
// columns of the dense row B[col, :] (coalesced 32*NPL-wide reads).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace rsvd {

namespace {

template <typename T, typename I, int NPL>
__global__ void __launch_bounds__(256)
k_spmm_csr(int64_t nrows, int64_t nb, const I* __restrict__ indptr, const I* __restrict__ col,
           const T* __restrict__ val, const T* __restrict__ B, int64_t ldb, double alpha,
           double beta, T* __restrict__ C, int64_t ldc) {
    const int lane = threadIdx.x & 31;
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= nrows) return;
    T acc[NPL];
#pragma unroll
    for (int t = 0; t < NPL; ++t) acc[t] = T(0);
    const int64_t lo = (int64_t)indptr[row], hi = (int64_t)indptr[row + 1];
    for (int64_t base = lo; base < hi; base += 32) {
        const int64_t e = base + lane;
        int64_t c = 0;
        T v = T(0);
        if (e < hi) {
            c = (int64_t)col[e];
            v = val[e];
        }
        const int cnt = (int)min((int64_t)32, hi - base);
        for (int i = 0; i < cnt; ++i) {
            const int64_t ci = __shfl_sync(0xffffffffu, c, i);
            const T vi = __shfl_sync(0xffffffffu, v, i);
            const T* brow = B + ci * ldb;
#pragma unroll
            for (int t = 0; t < NPL; ++t) {
                const int64_t j = lane + 32 * t;
                if (j < nb) acc[t] = fma(vi, brow[j], acc[t]);
            }
        }
    }
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
        const int64_t j = lane + 32 * t;
        if (j < nb) {
            double r = alpha * (double)acc[t];
            if (beta != 0.0) r += beta * (double)C[row * ldc + j];
            C[row * ldc + j] = (T)r;
        }
    }
}

template <typename T, typename I>
int launch_spmm(int64_t nrows, int64_t nb, const void* indptr, const void* col, const void* val,
                const void* B, int64_t ldb, double alpha, double beta, void* C, int64_t ldc,
                cudaStream_t st) {
    unsigned grid = (unsigned)cdiv(nrows * 32, 256);
    const I* ip = (const I*)indptr;
    const I* cp = (const I*)col;
    const T* vp = (const T*)val;
    const T* bp = (const T*)B;
    T* cc = (T*)C;
    if (nb <= 32)
        k_spmm_csr<T, I, 1><<<grid, 256, 0, st>>>(nrows, nb, ip, cp, vp, bp, ldb, alpha, beta, cc, ldc);
    else if (nb <= 64)
        k_spmm_csr<T, I, 2><<<grid, 256, 0, st>>>(nrows, nb, ip, cp, vp, bp, ldb, alpha, beta, cc, ldc);
    else if (nb <= 128)
        k_spmm_csr<T, I, 4><<<grid, 256, 0, st>>>(nrows, nb, ip, cp, vp, bp, ldb, alpha, beta, cc, ldc);
    else if (nb <= 256)
        k_spmm_csr<T, I, 8><<<grid, 256, 0, st>>>(nrows, nb, ip, cp, vp, bp, ldb, alpha, beta, cc, ldc);
    else {
        // wide blocks: process in column panels of 256
        for (int64_t j0 = 0; j0 < nb; j0 += 256) {
            int64_t w = nb - j0 < 256 ? nb - j0 : 256;
            k_spmm_csr<T, I, 8><<<grid, 256, 0, st>>>(nrows, w, ip, cp, vp, bp + j0, ldb, alpha,
                                                       beta, cc + j0, ldc);
        }
    }
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

// ---------------------------------------------------------------------------
// Load-balanced product with a row-split plan (built once per operator): a
// chunk is (row, nonzeros [lo, hi), slot). Rows of at most `chunk` nonzeros
// are one chunk written straight to C (slot -1); longer rows (the Zipf
// columns of A^T: 194k nonzeros in C3's column 0) are cut into chunks whose
// partial sums go to workspace slots and are added in chunk order by
// k_spmm_split_reduce (deterministic). Warp per chunk; 4 nonzeros in flight
// per lane; FP32 rows of B gathered as float4 (VEC) when aligned.
#ifndef RSVD_SPMM_UNROLL
#define RSVD_SPMM_UNROLL 4
#endif
#ifndef RSVD_SPMM_MINB
#define RSVD_SPMM_MINB 1
#endif
template <typename T, typename I, int NPL, bool VEC>
__global__ void __launch_bounds__(256, RSVD_SPMM_MINB)
k_spmm_plan(int64_t nchunks, int64_t nb, const I* __restrict__ col, const T* __restrict__ val,
            const T* __restrict__ B, int64_t ldb, double alpha, double beta, T* __restrict__ C, int64_t ldc,
            const int64_t* __restrict__ clo, const int64_t* __restrict__ chi, const int32_t* __restrict__ crow,
            const int32_t* __restrict__ cslot, T* __restrict__ ws) {
    const int lane = threadIdx.x & 31;
    const int64_t ch = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (ch >= nchunks) return;
    constexpr int W = VEC ? 4 * NPL : NPL;  // outputs per lane
    T acc[W];
#pragma unroll
    for (int t = 0; t < W; ++t) acc[t] = T(0);
    const int64_t lo = clo[ch], hi = chi[ch];
    auto accum = [&](const T* brow, T v) {
        if constexpr (VEC) {
#pragma unroll
            for (int t = 0; t < NPL; ++t) {
                const int64_t j = 4 * (lane + 32 * t);
                if (j < nb) {
                    const float4 b4 = *reinterpret_cast<const float4*>(brow + j);
                    acc[4 * t + 0] = fmaf(v, b4.x, acc[4 * t + 0]);
                    acc[4 * t + 1] = fmaf(v, b4.y, acc[4 * t + 1]);
                    acc[4 * t + 2] = fmaf(v, b4.z, acc[4 * t + 2]);
                    acc[4 * t + 3] = fmaf(v, b4.w, acc[4 * t + 3]);
                }
            }
        } else {
#pragma unroll
            for (int t = 0; t < NPL; ++t) {
                const int64_t j = lane + 32 * t;
                if (j < nb) acc[t] = fma(v, brow[j], acc[t]);
            }
        }
    };
    for (int64_t base = lo; base < hi; base += 32) {
        const int64_t e = base + lane;
        int64_t c = 0;
        T v = T(0);
        if (e < hi) {
            c = (int64_t)col[e];
            v = val[e];
        }
        const int cnt = (int)min((int64_t)32, hi - base);
        int i = 0;
        constexpr int U = RSVD_SPMM_UNROLL;  // nonzeros (row gathers) in flight per warp
        for (; i + U <= cnt; i += U) {
            int64_t cu[U];
            T vu[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                cu[u] = __shfl_sync(0xffffffffu, c, i + u);
                vu[u] = __shfl_sync(0xffffffffu, v, i + u);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) accum(B + cu[u] * ldb, vu[u]);
        }
        for (; i < cnt; ++i) {
            const int64_t ci = __shfl_sync(0xffffffffu, c, i);
            const T vi = __shfl_sync(0xffffffffu, v, i);
            accum(B + ci * ldb, vi);
        }
    }
    const int slot = cslot[ch];
    const int64_t row = crow[ch];
#pragma unroll
    for (int t = 0; t < W; ++t) {
        const int64_t j = VEC ? 4 * (lane + 32 * (t / 4)) + (t % 4) : lane + 32 * t;
        if (j >= nb) continue;
        if (slot >= 0) {
            ws[(int64_t)slot * nb + j] = acc[t];
        } else {
            double r = alpha * (double)acc[t];
            if (beta != 0.0) r += beta * (double)C[row * ldc + j];
            C[row * ldc + j] = (T)r;
        }
    }
}

// FP32 / int32 / width <= 128 (a multiple of 4) fast path of the plan product:
// persistent warps (chunks w, w + W, ...: no CTA launch churn, no CTA held by
// its longest row), U row gathers in flight per lane with the batch padded to
// a multiple of U by (column 0, value 0) entries instead of a remainder loop,
// 32-bit column shuffles. ncu of k_spmm_plan on C3's cold CSR: 27.7
// instructions per nonzero, 19 of 64 warps resident on average, 5.7-7 TB/s of
// gathered rows against the 12-16 TB/s a bare gather loop reaches
// (tools/l2_gather_probe.cu).
template <int U>
__global__ void __launch_bounds__(256, 3)
k_spmm_gather_f32(int64_t nchunks, int nb, const int32_t* __restrict__ col, const float* __restrict__ val,
                  const float* __restrict__ B, int64_t ldb, float alpha, float beta, float* __restrict__ C,
                  int64_t ldc, const int64_t* __restrict__ clo, const int64_t* __restrict__ chi,
                  const int32_t* __restrict__ crow, const int32_t* __restrict__ cslot, float* __restrict__ ws) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool on = 4 * lane < nb;
    const float* Bl = B + 4 * lane;
    for (int64_t ch = gw; ch < nchunks; ch += nwarps) {
        const int64_t lo = clo[ch], hi = chi[ch];
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t base = lo; base < hi; base += 32) {
            const int64_t e = base + lane;
            int c = 0;
            float v = 0.f;
            if (e < hi) {
                c = col[e];
                v = val[e];
            }
            const int cnt = (int)min((int64_t)32, hi - base);
            for (int i = 0; i < cnt; i += U) {
                int cu[U];
                float vu[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    cu[u] = __shfl_sync(0xffffffffu, c, i + u);
                    vu[u] = __shfl_sync(0xffffffffu, v, i + u);
                }
                float4 b4[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    b4[u] = on ? *reinterpret_cast<const float4*>(Bl + (int64_t)cu[u] * ldb)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    acc.x = fmaf(vu[u], b4[u].x, acc.x);
                    acc.y = fmaf(vu[u], b4[u].y, acc.y);
                    acc.z = fmaf(vu[u], b4[u].z, acc.z);
                    acc.w = fmaf(vu[u], b4[u].w, acc.w);
                }
            }
        }
        if (!on) continue;
        const int slot = cslot[ch];
        if (slot >= 0) {
            *reinterpret_cast<float4*>(ws + (int64_t)slot * nb + 4 * lane) = acc;
        } else {
            float* cp = C + (int64_t)crow[ch] * ldc + 4 * lane;
            // same rounding as k_spmm_plan: alpha / beta applied in FP64
            float4 r;
            if (beta != 0.f) {
                const float4 o = *reinterpret_cast<const float4*>(cp);
                r.x = (float)((double)alpha * (double)acc.x + (double)beta * (double)o.x);
                r.y = (float)((double)alpha * (double)acc.y + (double)beta * (double)o.y);
                r.z = (float)((double)alpha * (double)acc.z + (double)beta * (double)o.z);
                r.w = (float)((double)alpha * (double)acc.w + (double)beta * (double)o.w);
            } else {
                r.x = (float)((double)alpha * (double)acc.x);
                r.y = (float)((double)alpha * (double)acc.y);
                r.z = (float)((double)alpha * (double)acc.z);
                r.w = (float)((double)alpha * (double)acc.w);
            }
            *reinterpret_cast<float4*>(cp) = r;
        }
    }
}

// Nonzero-balanced FP32 product (the default plan for FP32 / int32 / width <=
// 128): a work unit is a fixed run of `chunk` consecutive nonzeros, whatever
// rows they belong to. Measured on C3's cold CSR (tools/spmm_uniform_probe.py):
// warp-per-row reaches 10.5 TB/s of gathered rows when every row has 54
// nonzeros but 7.0 TB/s with C3's lognormal row lengths and the same columns
// -- the short rows' fixed cost (pointer loads, a gather tail that cannot fill
// the U loads in flight, the C row write) sets the pace, not the column
// pattern. Here a warp walks its run 32 nonzeros at a time with U row gathers
// in flight; at a row change it flushes the finished row: straight to C when
// the row lies inside the run, to a workspace slot when it is the run's first
// or last row and continues in a neighbouring run (head_slot / tail_slot from
// the plan; a row's slots are consecutive and k_spmm_split_reduce adds them in
// order: deterministic, no atomics). Rows without nonzeros are scaled by
// k_spmm_empty_rows.
#ifndef RSVD_SPMM_NNZ_MINB
#define RSVD_SPMM_NNZ_MINB 3
#endif
template <int U>
__global__ void __launch_bounds__(256, U >= 16 ? 2 : RSVD_SPMM_NNZ_MINB)
k_spmm_nnz_f32(int64_t nnz, int chunk, int64_t nchunks, int nb, const int32_t* __restrict__ col,
               const float* __restrict__ val, const int32_t* __restrict__ rowid, const float* __restrict__ B,
               int64_t ldb, float alpha, float beta, float* __restrict__ C, int64_t ldc,
               const int32_t* __restrict__ head_slot, const int32_t* __restrict__ tail_slot,
               float* __restrict__ ws, int ablate) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool on = 4 * lane < nb;
    const float* Bl = B + 4 * lane;
    for (int64_t ch = gw; ch < nchunks; ch += nwarps) {
        const int64_t e0 = ch * chunk, e1 = min(nnz, e0 + (int64_t)chunk);
        const int hs = head_slot[ch], ts = tail_slot[ch];
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        int cur = -1;
        bool first = true;  // the row being accumulated is the run's first row
        auto flush = [&](bool last) {
            if (!on) return;
            if ((ablate & 1) && acc.x != 1234.5f) return;  // profiling: no stores
            const int slot = first ? hs : (last ? ts : -1);
            if (slot >= 0) {
                *reinterpret_cast<float4*>(ws + (int64_t)slot * nb + 4 * lane) = acc;
            } else {
                float* cp = C + (int64_t)cur * ldc + 4 * lane;
                float4 r;
                if (beta != 0.f) {
                    const float4 o = *reinterpret_cast<const float4*>(cp);
                    r.x = (float)((double)alpha * (double)acc.x + (double)beta * (double)o.x);
                    r.y = (float)((double)alpha * (double)acc.y + (double)beta * (double)o.y);
                    r.z = (float)((double)alpha * (double)acc.z + (double)beta * (double)o.z);
                    r.w = (float)((double)alpha * (double)acc.w + (double)beta * (double)o.w);
                } else {
                    r.x = (float)((double)alpha * (double)acc.x);
                    r.y = (float)((double)alpha * (double)acc.y);
                    r.z = (float)((double)alpha * (double)acc.z);
                    r.w = (float)((double)alpha * (double)acc.w);
                }
                *reinterpret_cast<float4*>(cp) = r;
            }
        };
        for (int64_t base = e0; base < e1; base += 32) {
            const int64_t e = base + lane;
            const int cnt = (int)min((int64_t)32, e1 - base);
            int c = 0, r = 0;
            float v = 0.f;
            if (e < e1) {
                c = col[e];
                v = (ablate & 4) ? 1.f : val[e];
                r = (ablate & 2) ? 0 : rowid[e];
            }
            // padding entries (value 0, column 0) stay in the batch's last row
            const int r_last = __shfl_sync(0xffffffffu, r, cnt - 1);  // every lane takes part in the shuffle
            r = lane < cnt ? r : r_last;
            // row starts of the batch as a bit mask: a group of U gathers without a
            // start runs the bare FMA loop (no row-id shuffles, no branches between the
            // FMAs: 85 % of the groups at C3's ~54 nonzeros per row; the probe's loop
            // loses 22 % to per-nonzero row bookkeeping)
            int prev = __shfl_up_sync(0xffffffffu, r, 1);
            if (lane == 0) prev = cur;
            const unsigned starts = __ballot_sync(0xffffffffu, r != prev);
            for (int i = 0; i < cnt; i += U) {
                int cu[U];
                float vu[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    cu[u] = __shfl_sync(0xffffffffu, c, i + u);
                    vu[u] = __shfl_sync(0xffffffffu, v, i + u);
                }
                float4 b4[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    b4[u] = on ? *reinterpret_cast<const float4*>(Bl + (int64_t)cu[u] * ldb)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
                const unsigned gm = (starts >> i) & ((1u << U) - 1u);
                if (gm == 0u) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        acc.x = fmaf(vu[u], b4[u].x, acc.x);
                        acc.y = fmaf(vu[u], b4[u].y, acc.y);
                        acc.z = fmaf(vu[u], b4[u].z, acc.z);
                        acc.w = fmaf(vu[u], b4[u].w, acc.w);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if ((gm >> u) & 1u) {  // warp-uniform: entry i + u opens a row
                            if (cur >= 0) {
                                flush(false);
                                first = false;
                            }
                            cur = __shfl_sync(0xffffffffu, r, i + u);
                            acc = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                        acc.x = fmaf(vu[u], b4[u].x, acc.x);
                        acc.y = fmaf(vu[u], b4[u].y, acc.y);
                        acc.z = fmaf(vu[u], b4[u].z, acc.z);
                        acc.w = fmaf(vu[u], b4[u].w, acc.w);
                    }
                }
            }
        }
        if (cur >= 0) flush(true);
    }
}

// rows without a nonzero: C[r, :] = beta C[r, :]
__global__ void k_spmm_empty_rows(int64_t nempty, int nb, const int32_t* __restrict__ rows, float beta,
                                  float* __restrict__ C, int64_t ldc) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nempty * nb) return;
    const int64_t i = e / nb, j = e % nb;
    float* p = C + (int64_t)rows[i] * ldc + j;
    *p = beta != 0.f ? beta * *p : 0.f;
}

template <typename T>
__global__ void k_spmm_split_reduce(int64_t nsplit, int64_t nb, const int32_t* __restrict__ srow,
                                    const int64_t* __restrict__ sbeg, const T* __restrict__ ws, double alpha,
                                    double beta, T* __restrict__ C, int64_t ldc) {
    const int lane = threadIdx.x & 31;
    const int64_t sidx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (sidx >= nsplit) return;
    const int64_t row = srow[sidx], b0 = sbeg[sidx], b1 = sbeg[sidx + 1];
    for (int64_t j = lane; j < nb; j += 32) {
        double acc = 0.0;
        for (int64_t sl = b0; sl < b1; ++sl) acc += (double)ws[sl * nb + j];
        double r = alpha * acc;
        if (beta != 0.0) r += beta * (double)C[row * ldc + j];
        C[row * ldc + j] = (T)r;
    }
}

template <typename T, typename I>
int launch_spmm_plan_panel(int64_t nb, const void* col, const void* val, const T* bp, int64_t ldb, double alpha,
                           double beta, T* cc, int64_t ldc, int64_t nchunks, const int64_t* clo, const int64_t* chi,
                           const int32_t* crow, const int32_t* cslot, int64_t nsplit, const int32_t* srow,
                           const int64_t* sbeg, void* ws, cudaStream_t st) {
    const unsigned grid = (unsigned)cdiv(nchunks * 32, 256);
    const I* cp = (const I*)col;
    const T* vp = (const T*)val;
    T* wp = (T*)ws;
    const bool vec = sizeof(T) == 4 && ldb % 4 == 0 && nb % 4 == 0 && ((uintptr_t)bp & 15) == 0;
    if constexpr (sizeof(T) == 4 && sizeof(I) == 4) {
        // persistent fast path (RSVD_SPMM_OLD=1: k_spmm_plan, for A/B measurement);
        // C rows and workspace slots must take float4 stores
        static const bool old_path = getenv("RSVD_SPMM_OLD") != nullptr;
        static const int unroll = getenv("RSVD_SPMM_U") ? atoi(getenv("RSVD_SPMM_U")) : 8;
        if (!old_path && vec && nb <= 128 && nchunks > 0 && ldc % 4 == 0 && ((uintptr_t)cc & 15) == 0 &&
            ((uintptr_t)wp & 15) == 0) {
            const int64_t want = cdiv(nchunks * 32, 256);
            const unsigned g = (unsigned)std::min<int64_t>(want, (int64_t)sm_count() * 3);
            if (unroll == 4)
                k_spmm_gather_f32<4><<<g, 256, 0, st>>>(nchunks, (int)nb, (const int32_t*)cp, (const float*)vp,
                                                        (const float*)bp, ldb, (float)alpha, (float)beta, (float*)cc,
                                                        ldc, clo, chi, crow, cslot, (float*)wp);
            else
                k_spmm_gather_f32<8><<<g, 256, 0, st>>>(nchunks, (int)nb, (const int32_t*)cp, (const float*)vp,
                                                        (const float*)bp, ldb, (float)alpha, (float)beta, (float*)cc,
                                                        ldc, clo, chi, crow, cslot, (float*)wp);
            RSVD_CHECK_LAUNCH();
            if (nsplit > 0) {
                k_spmm_split_reduce<T><<<(unsigned)cdiv(nsplit * 32, 256), 256, 0, st>>>(nsplit, nb, srow, sbeg, wp,
                                                                                         alpha, beta, cc, ldc);
                RSVD_CHECK_LAUNCH();
            }
            return RSVD_OK;
        }
    }
    if (nchunks > 0) {
        if (vec && nb <= 128)
            k_spmm_plan<T, I, 1, true><<<grid, 256, 0, st>>>(nchunks, nb, cp, vp, bp, ldb, alpha, beta, cc, ldc, clo,
                                                              chi, crow, cslot, wp);
        else if (vec && nb <= 256)
            k_spmm_plan<T, I, 2, true><<<grid, 256, 0, st>>>(nchunks, nb, cp, vp, bp, ldb, alpha, beta, cc, ldc, clo,
                                                              chi, crow, cslot, wp);
        else if (nb <= 32)
            k_spmm_plan<T, I, 1, false><<<grid, 256, 0, st>>>(nchunks, nb, cp, vp, bp, ldb, alpha, beta, cc, ldc,
                                                               clo, chi, crow, cslot, wp);
        else if (nb <= 64)
            k_spmm_plan<T, I, 2, false><<<grid, 256, 0, st>>>(nchunks, nb, cp, vp, bp, ldb, alpha, beta, cc, ldc,
                                                               clo, chi, crow, cslot, wp);
        else if (nb <= 128)
            k_spmm_plan<T, I, 4, false><<<grid, 256, 0, st>>>(nchunks, nb, cp, vp, bp, ldb, alpha, beta, cc, ldc,
                                                               clo, chi, crow, cslot, wp);
        else
            k_spmm_plan<T, I, 8, false><<<grid, 256, 0, st>>>(nchunks, nb, cp, vp, bp, ldb, alpha, beta, cc, ldc,
                                                               clo, chi, crow, cslot, wp);
        RSVD_CHECK_LAUNCH();
    }
    if (nsplit > 0) {
        k_spmm_split_reduce<T><<<(unsigned)cdiv(nsplit * 32, 256), 256, 0, st>>>(nsplit, nb, srow, sbeg, wp, alpha,
                                                                                 beta, cc, ldc);
        RSVD_CHECK_LAUNCH();
    }
    return RSVD_OK;
}

// wide blocks run in column panels of 256 (the workspace holds one panel's
// partials; panels are stream-ordered)
template <typename T, typename I>
int launch_spmm_plan(int64_t nb, const void* col, const void* val, const void* B, int64_t ldb, double alpha,
                     double beta, void* C, int64_t ldc, int64_t nchunks, const int64_t* clo, const int64_t* chi,
                     const int32_t* crow, const int32_t* cslot, int64_t nsplit, const int32_t* srow,
                     const int64_t* sbeg, void* ws, cudaStream_t st) {
    for (int64_t j0 = 0; j0 < nb; j0 += 256) {
        const int64_t wdt = nb - j0 < 256 ? nb - j0 : 256;
        const int rc = launch_spmm_plan_panel<T, I>(wdt, col, val, (const T*)B + j0, ldb, alpha, beta, (T*)C + j0,
                                                    ldc, nchunks, clo, chi, crow, cslot, nsplit, srow, sbeg, ws, st);
        if (rc) return rc;
    }
    return RSVD_OK;
}

// ---------------------------------------------------------------------------
// Slab tier of the hybrid product A X: the M most frequent columns that are
// too sparse for the dense panel (C3: density 0.2 % - 3 %, ~21 % of the
// nonzeros) keep their rows of the dense block X in SHARED MEMORY, so their
// nonzeros cost a 100-byte shared-memory read instead of a 400-byte L2 gather.
// The block width is cut into `nwc` column chunks of wb <= 32 floats so that
// M x wb x 4 bytes fit one SM (C3: width 100 -> 4 chunks of 25, M = 2048,
// 200 KB): CTA (g, wc) stages X[slab_cols, wc-th chunk] once and walks the
// rows of row group g, warp per row, lane per output column; every lane of a
// warp reads consecutive words of one slab row (conflict-free). The rows'
// slab nonzeros come from their own CSR (slab row index instead of the column
// index). C[r, chunk] += sum (fixed order: deterministic).
__global__ void __launch_bounds__(1024, 1)
k_spmm_slab(int64_t nrows, int64_t nb, int wb, int64_t rows_per_group, const int32_t* __restrict__ mptr,
            const int32_t* __restrict__ midx, const float* __restrict__ mval, const int64_t* __restrict__ slab_cols,
            int M, const float* __restrict__ X, int64_t ldx, float* __restrict__ C, int64_t ldc) {
    extern __shared__ float slab[];  // [M][wb]
    const int w0 = blockIdx.y * wb;
    const int wn = (int)min((int64_t)wb, nb - w0);  // live columns of this chunk
    for (int e = threadIdx.x; e < M * wb; e += blockDim.x) {
        const int sidx = e / wb, j = e - sidx * wb;
        slab[e] = j < wn ? X[slab_cols[sidx] * ldx + w0 + j] : 0.f;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_group;
    const int64_t r1 = min(nrows, r0 + rows_per_group);
    const bool live = lane < wn;
    const float* sl = slab + (live ? lane : 0);
    for (int64_t r = r0 + warp; r < r1; r += nw) {
        const int lo = mptr[r], hi = mptr[r + 1];
        if (lo == hi) continue;
        float acc0 = 0.f, acc1 = 0.f;
        for (int base = lo; base < hi; base += 32) {
            const int e = base + lane;
            int si = 0;
            float v = 0.f;
            if (e < hi) {
                si = midx[e] * wb;
                v = mval[e];
            }
            const int cnt = min(32, hi - base);
            int i = 0;
            for (; i + 2 <= cnt; i += 2) {
                const int s0 = __shfl_sync(0xffffffffu, si, i), s1 = __shfl_sync(0xffffffffu, si, i + 1);
                const float v0 = __shfl_sync(0xffffffffu, v, i), v1 = __shfl_sync(0xffffffffu, v, i + 1);
                acc0 = fmaf(v0, sl[s0], acc0);
                acc1 = fmaf(v1, sl[s1], acc1);
            }
            if (i < cnt) {
                const int s0 = __shfl_sync(0xffffffffu, si, i);
                const float v0 = __shfl_sync(0xffffffffu, v, i);
                acc0 = fmaf(v0, sl[s0], acc0);
            }
        }
        if (live) C[r * ldc + w0 + lane] += acc0 + acc1;
    }
}

template <typename T, typename I>
__global__ void k_csr_transpose_fill(int64_t nrows, int64_t nnz, const I* __restrict__ indptr,
                                     const I* __restrict__ col, const T* __restrict__ val,
                                     const int64_t* __restrict__ perm, I* __restrict__ tcol,
                                     T* __restrict__ tval) {
    int64_t e2 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e2 >= nnz) return;
    int64_t e = perm[e2];
    // row of nonzero e: last r with indptr[r] <= e
    int64_t lo = 0, hi = nrows;  // indptr[lo] <= e < indptr[hi]
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if ((int64_t)indptr[mid] <= e) lo = mid;
        else hi = mid;
    }
    tcol[e2] = (I)lo;
    tval[e2] = val[e];
}

template <typename I>
__global__ void k_csr_transpose_ptr(int64_t ncols, int64_t nnz, const I* __restrict__ col,
                                    const int64_t* __restrict__ perm, I* __restrict__ tptr) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncols) return;
    // first position e2 with col[perm[e2]] >= c
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((int64_t)col[perm[mid]] < c) lo = mid + 1;
        else hi = mid;
    }
    tptr[c] = (I)lo;
}

}  // namespace

int spmm_csr(int dtype, int idx64, int64_t nrows, int64_t ncols, int64_t nb, const void* indptr,
             const void* col, const void* val, const void* B, int64_t ldb, double alpha,
             double beta, void* C, int64_t ldc, cudaStream_t st) {
    (void)ncols;
    if (nrows == 0 || nb == 0) return RSVD_OK;
    if (dtype == RSVD_F64)
        return idx64 ? launch_spmm<double, int64_t>(nrows, nb, indptr, col, val, B, ldb, alpha, beta, C, ldc, st)
                     : launch_spmm<double, int32_t>(nrows, nb, indptr, col, val, B, ldb, alpha, beta, C, ldc, st);
    return idx64 ? launch_spmm<float, int64_t>(nrows, nb, indptr, col, val, B, ldb, alpha, beta, C, ldc, st)
                 : launch_spmm<float, int32_t>(nrows, nb, indptr, col, val, B, ldb, alpha, beta, C, ldc, st);
}

int spmm_csr_plan(int dtype, int idx64, int64_t nb, const void* col, const void* val, const void* B, int64_t ldb,
                  double alpha, double beta, void* C, int64_t ldc, int64_t nchunks, const int64_t* clo,
                  const int64_t* chi, const int32_t* crow, const int32_t* cslot, int64_t nsplit,
                  const int32_t* srow, const int64_t* sbeg, void* ws, cudaStream_t st) {
    if (nb == 0) return RSVD_OK;
#define RSVD_SPP(T, I)                                                                                          \
    return launch_spmm_plan<T, I>(nb, col, val, B, ldb, alpha, beta, C, ldc, nchunks, clo, chi, crow, cslot, \
                                  nsplit, srow, sbeg, ws, st)
    if (dtype == RSVD_F64) {
        if (idx64) RSVD_SPP(double, int64_t);
        RSVD_SPP(double, int32_t);
    }
    if (idx64) RSVD_SPP(float, int64_t);
    RSVD_SPP(float, int32_t);
#undef RSVD_SPP
}

int spmm_slab(int64_t nrows, int64_t nb, const int32_t* mptr, const int32_t* midx, const float* mval,
              const int64_t* slab_cols, int64_t M, const float* X, int64_t ldx, float* C, int64_t ldc,
              cudaStream_t st) {
    if (nrows == 0 || nb == 0 || M == 0) return RSVD_OK;
    // chunks of wb <= 32 columns whose M-row slab fits 200 KB of shared memory
    const int64_t cap = 200 * 1024;
    int64_t nwc = cdiv(nb, 32);
    while (M * cdiv(nb, nwc) * 4 > cap) ++nwc;
    const int wb = (int)cdiv(nb, nwc);
    nwc = cdiv(nb, wb);
    const size_t sm = (size_t)M * wb * sizeof(float);
    static PerDevice<bool> attr_dev;
    bool& attr = attr_dev.get();
    if (!attr) {
        RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_spmm_slab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap));
        attr = true;
    }
    // one CTA per SM: row groups x width chunks
    int64_t groups = sm_count() / nwc;
    if (groups < 1) groups = 1;
    const int64_t rpg = cdiv(nrows, groups);
    groups = cdiv(nrows, rpg);
    dim3 grid((unsigned)groups, (unsigned)nwc);
    k_spmm_slab<<<grid, 1024, sm, st>>>(nrows, nb, wb, rpg, mptr, midx, mval, slab_cols, (int)M, X, ldx, C, ldc);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int spmm_nnz_plan(int64_t nnz, int chunk, int64_t nb, const int32_t* col, const float* val, const int32_t* rowid,
                  const float* B, int64_t ldb, double alpha, double beta, float* C, int64_t ldc,
                  const int32_t* head_slot, const int32_t* tail_slot, int64_t nsplit, const int32_t* srow,
                  const int64_t* sbeg, int64_t nempty, const int32_t* empty_rows, float* ws, cudaStream_t st) {
    if (nb == 0) return RSVD_OK;
    RSVD_REQUIRE(nb <= 128 && nb % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 && ((uintptr_t)B & 15) == 0 &&
                     ((uintptr_t)C & 15) == 0 && ((uintptr_t)ws & 15) == 0,
                 "spmm_nnz_plan: width <= 128, a multiple of 4, 16-byte aligned rows");
    RSVD_REQUIRE(chunk >= 32 && chunk % 32 == 0, "spmm_nnz_plan: chunk must be a multiple of 32");
    const int64_t nchunks = cdiv(nnz, chunk);
    if (nchunks > 0) {
        static const int ctas = getenv("RSVD_SPMM_CTAS") ? atoi(getenv("RSVD_SPMM_CTAS")) : 3;
        const unsigned g = (unsigned)std::min<int64_t>(cdiv(nchunks * 32, 256), (int64_t)sm_count() * ctas);
        static const int unroll = getenv("RSVD_SPMM_U") ? atoi(getenv("RSVD_SPMM_U")) : 8;
        static const int abl = getenv("RSVD_SPMM_ABLATE") ? atoi(getenv("RSVD_SPMM_ABLATE")) : 0;
        if (unroll == 4)
            k_spmm_nnz_f32<4><<<g, 256, 0, st>>>(nnz, chunk, nchunks, (int)nb, col, val, rowid, B, ldb, (float)alpha,
                                                 (float)beta, C, ldc, head_slot, tail_slot, ws, abl);
        else if (unroll == 16)
            k_spmm_nnz_f32<16><<<g, 256, 0, st>>>(nnz, chunk, nchunks, (int)nb, col, val, rowid, B, ldb, (float)alpha,
                                                  (float)beta, C, ldc, head_slot, tail_slot, ws, abl);
        else
            k_spmm_nnz_f32<8><<<g, 256, 0, st>>>(nnz, chunk, nchunks, (int)nb, col, val, rowid, B, ldb, (float)alpha,
                                                 (float)beta, C, ldc, head_slot, tail_slot, ws, abl);
        RSVD_CHECK_LAUNCH();
    }
    if (nsplit > 0) {
        k_spmm_split_reduce<float><<<(unsigned)cdiv(nsplit * 32, 256), 256, 0, st>>>(nsplit, nb, srow, sbeg, ws, alpha,
                                                                                     beta, C, ldc);
        RSVD_CHECK_LAUNCH();
    }
    if (nempty > 0) {
        k_spmm_empty_rows<<<(unsigned)cdiv(nempty * nb, 256), 256, 0, st>>>(nempty, (int)nb, empty_rows, (float)beta, C,
                                                                            ldc);
        RSVD_CHECK_LAUNCH();
    }
    return RSVD_OK;
}

template <typename T, typename I>
static int csr_t(int64_t nrows, int64_t ncols, int64_t nnz, const void* indptr, const void* col,
                 const void* val, const int64_t* perm, void* tptr, void* tcol, void* tval,
                 cudaStream_t st) {
    if (nnz > 0) {
        k_csr_transpose_fill<T, I><<<(unsigned)cdiv(nnz, 256), 256, 0, st>>>(
            nrows, nnz, (const I*)indptr, (const I*)col, (const T*)val, perm, (I*)tcol, (T*)tval);
        RSVD_CHECK_LAUNCH();
    }
    k_csr_transpose_ptr<I><<<(unsigned)cdiv(ncols + 1, 256), 256, 0, st>>>(
        ncols, nnz, (const I*)col, perm, (I*)tptr);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int csr_transpose(int dtype, int idx64, int64_t nrows, int64_t ncols, int64_t nnz,
                  const void* indptr, const void* col, const void* val, const int64_t* perm,
                  void* tptr, void* tcol, void* tval, cudaStream_t st) {
    if (dtype == RSVD_F64)
        return idx64 ? csr_t<double, int64_t>(nrows, ncols, nnz, indptr, col, val, perm, tptr, tcol, tval, st)
                     : csr_t<double, int32_t>(nrows, ncols, nnz, indptr, col, val, perm, tptr, tcol, tval, st);
    return idx64 ? csr_t<float, int64_t>(nrows, ncols, nnz, indptr, col, val, perm, tptr, tcol, tval, st)
                 : csr_t<float, int32_t>(nrows, ncols, nnz, indptr, col, val, perm, tptr, tcol, tval, st);
}

}  // namespace rsvd
