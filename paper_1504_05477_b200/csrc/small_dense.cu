// Small dense FP64 kernels of the orthonormalization and the Rayleigh-Ritz
// eigensolve.
//
//  * chol_deflate: column-ordered Cholesky of a block Gram with deficiency
//    deflation + the inverse triangular factor. Together with two GEMMs this
//    is the blocked replacement of the per-column CGS2 loop of _mgs
//    (factor.py:79-118): same column order, same "residual small relative to
//    the original column norm" test (factor.py:105), same fill stream for the
//    replaced columns (factor.py:89-90, 107).
//  * jacobi: two-sided Jacobi with the reference's stop and skip rules
//    (_kernels.pyx:127-192) in round-robin ("circle method") parallel order,
//    as ONE cooperative persistent kernel: per round every CTA recomputes the
//    W2/2 rotations of the round from the diagonal/pair entries, applies
//    M' = J^T M J blockwise (2x2 blocks are independent) and V' = V J, and
//    writes the result in the NEXT round's slot order (ping-pong buffers), so
//    every round's pairs are adjacent (2i, 2i+1) and loads stay coalesced.
//    After a whole sweep (W2-1 rounds) the slot order is the identity again.
//  * eig_select: descending stable sort of the eigenvalues (factor.py:164-165)
//    and gather of the top-k eigenvectors.
#include <cooperative_groups.h>

#include "common.cuh"

namespace rsvd {

namespace {

// ---------------------------------------------------------------------------
// chol_deflate
__device__ __forceinline__ int64_t tri_off(int64_t p, int64_t i, int64_t j) {
    // packed upper triangle, row-major, i <= j
    return i * p - (i * (i - 1)) / 2 + (j - i);
}

constexpr int kCholThreads = 256;
constexpr int kMaxSmemP = 512;

// One CTA. R (upper triangle, packed) lives in shared memory; T = R^{-1} in
// shared memory too when it fits (else it is built in place in global T).
// Right-looking Cholesky (p sequential column steps), then T by rows from
// the bottom: T[a][c] = -(sum_{b=a+1..c} R[a][b] T[b][c]) / R[a][a], all c in
// parallel per row a.
__global__ void __launch_bounds__(kCholThreads)
k_chol_deflate(int64_t p, const double* __restrict__ G, int64_t ldg,
               const double* __restrict__ ref2, double tau2, double* __restrict__ T, int64_t ldt,
               int32_t* __restrict__ mask, int32_t* __restrict__ ndef, int32_t* __restrict__ running,
               const int32_t* __restrict__ active, double* gws, int use_smem, int t_in_smem,
               const int32_t* __restrict__ pred) {
    if (pred && *pred == 0) return;
    extern __shared__ double smem_d[];
    double* S = use_smem ? smem_d : gws;
    const int64_t tri = p * (p + 1) / 2;
    double* Ts = t_in_smem ? smem_d + tri : nullptr;
    const int64_t ldT = t_in_smem ? p : ldt;
    double* Tw = t_in_smem ? Ts : T;
    __shared__ int s_def;
    __shared__ int s_count;
    __shared__ double s_rjj;
    __shared__ double s_ref[kMaxSmemP];
    __shared__ int s_act[kMaxSmemP];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const bool small = p <= kMaxSmemP;
    for (int64_t i = warp; i < p; i += nwarps)
        for (int64_t j = i + lane; j < p; j += 32) S[tri_off(p, i, j)] = G[i * ldg + j];
    if (small)
        for (int64_t j = tid; j < p; j += blockDim.x) {  // per-column inputs staged once
            s_ref[j] = ref2 ? ref2[j] : G[j * ldg + j];
            s_act[j] = active ? active[j] : 1;
        }
    if (tid == 0) s_count = 0;
    __syncthreads();
    for (int64_t j = 0; j < p; ++j) {
        if (tid == 0) {
            const double d = S[tri_off(p, j, j)];
            const double r = small ? s_ref[j] : (ref2 ? ref2[j] : G[j * ldg + j]);
            const int act = small ? s_act[j] : (active ? active[j] : 1);
            const int def = !act || !(d > tau2 * r) || !(d > 0.0);
            s_def = def;
            mask[j] = def ? (act ? 1 : 2) : 0;  // 2 = inactive slot (not counted)
            if (def && act) ++s_count;
            const double rjj = def ? 1.0 : sqrt(d);
            s_rjj = rjj;
            S[tri_off(p, j, j)] = rjj;
        }
        __syncthreads();
        const int def = s_def;
        const double inv = 1.0 / s_rjj;
        for (int64_t c = j + 1 + tid; c < p; c += blockDim.x) {
            const int64_t o = tri_off(p, j, c);
            S[o] = def ? 0.0 : S[o] * inv;
        }
        __syncthreads();
        if (!def) {
            // trailing update of the packed upper triangle, warp per row
            for (int64_t a = j + 1 + warp; a < p; a += nwarps) {
                const double ra = S[tri_off(p, j, a)];
                const int64_t rowa = tri_off(p, a, a) - a, rowj = tri_off(p, j, 0);
                for (int64_t b = a + lane; b < p; b += 32) S[rowa + b] -= ra * S[rowj + b];
            }
            __syncthreads();
        }
    }
    // T = R^{-1}, rows from the bottom
    for (int64_t a = p - 1; a >= 0; --a) {
        const double raa = S[tri_off(p, a, a)];
        const int64_t rowa = tri_off(p, a, a) - a;
        for (int64_t c = tid; c < p; c += blockDim.x) {
            double v;
            if (c < a) {
                v = 0.0;
            } else if (c == a) {
                v = 1.0 / raa;
            } else {
                double acc = 0.0;
                for (int64_t b = a + 1; b <= c; ++b) acc += S[rowa + b] * Tw[b * ldT + c];
                v = -acc / raa;
            }
            Tw[a * ldT + c] = v;
        }
        __syncthreads();
    }
    // zero row+column of deficient / inactive slots (rows already e_j), copy out
    for (int64_t e = tid; e < p * p; e += blockDim.x) {
        const int64_t i = e / p, c = e % p;
        double v = Tw[i * ldT + c];
        if (mask[i] || mask[c]) v = 0.0;
        T[i * ldt + c] = v;
    }
    __syncthreads();
    if (tid == 0) {
        const int32_t base = running ? running[0] : 0;
        ndef[0] = s_count;
        ndef[1] = base;
        if (running) running[0] = base + s_count;
    }
    for (int64_t j = tid; j < p; j += blockDim.x)
        if (mask[j] == 2) mask[j] = 0;
}

// Fast path for p <= kFastP: the packed Schur complement lives in typed
// shared memory. Every thread evaluates the pivot test itself (no serial
// thread-0 step), so a column costs one barrier; R's rows are scaled in one
// pass at the end. T = R^{-1} is built by ROWS (row c of T solves
// R^T s = e_c by forward substitution in axpy form), so every shared-memory
// access walks a row of the packed triangle (no bank conflicts); one warp
// per row, the row held in registers.
constexpr int kFastP = 224;

// ---------------------------------------------------------------------------
// Jacobi
constexpr int kJacThreads = 512;

struct JacobiState {
    int64_t n, W2;
    double* Mb[2];
    double* Vb[2];
    int64_t nv;  // rows of V
    double* partial;
    unsigned int* bar;
    double tol;
    int max_sweeps;
    int32_t* info;
    double* off_out;
};

__device__ __forceinline__ int64_t next_slot(int64_t s, int64_t W2) {
    if (W2 <= 2 || s == 0) return s;
    if ((s & 1) == 0) return (s == W2 - 2) ? W2 - 1 : s + 2;
    return (s == 1) ? 2 : s - 2;
}

// Deterministic grid-wide sum: fixed per-thread stride order, fixed block tree,
// fixed order over blocks. Every CTA returns the same value.
__device__ double grid_sum(double v, double* partial, unsigned int* bar) {
    __shared__ double red[kJacThreads / 32];
    __shared__ double total;
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
        partial[blockIdx.x] = s;
    }
    grid_barrier(bar, gridDim.x);
    if (threadIdx.x == 0) {
        volatile double* pv = partial;
        double s = 0.0;
        for (unsigned i = 0; i < gridDim.x; ++i) s += pv[i];
        total = s;
    }
    __syncthreads();
    double r = total;
    grid_barrier(bar, gridDim.x);  // partial[] reusable afterwards
    return r;
}

__global__ void __launch_bounds__(kJacThreads)
k_jacobi(JacobiState st) {
    extern __shared__ double sh[];
    const int64_t W2 = st.W2, n = st.n, half = W2 / 2;
    double* rc = sh;             // c per pair
    double* rs = sh + half;      // s per pair
    double* rt = sh + 2 * half;  // t per pair
    double* ra = sh + 3 * half;  // apq per pair
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;

    int cur = 0;
    // initial Frobenius norm and off-diagonal mass (reference order: fro, off)
    double fro2 = 0.0, off2 = 0.0;
    {
        const double* M = st.Mb[0];
        for (int64_t e = gtid; e < W2 * W2; e += gstride) {
            double x = M[e];
            fro2 += x * x;
            if (e / W2 != e % W2) off2 += x * x;
        }
    }
    const double fro = sqrt(grid_sum(fro2, st.partial, st.bar));
    double off = sqrt(grid_sum(off2, st.partial, st.bar));
    const double threshold = st.tol * fro;
    int sweeps = 0;
    bool converged = (n < 2) || (off <= threshold);
    const double skip = threshold * 1e-3 / (double)n;
    while (!converged && sweeps < st.max_sweeps) {
        for (int64_t round = 0; round < W2 - 1; ++round) {
            const double* M = st.Mb[cur];
            double* Mn = st.Mb[cur ^ 1];
            const double* V = st.Vb[cur];
            double* Vn = st.Vb[cur ^ 1];
            for (int64_t pr = threadIdx.x; pr < half; pr += blockDim.x) {
                const int64_t sp = 2 * pr, sq = 2 * pr + 1;
                const double apq = M[sp * W2 + sq];
                double c = 1.0, s = 0.0, t = 0.0;
                if (!(fabs(apq) <= skip)) {
                    const double app = M[sp * W2 + sp], aqq = M[sq * W2 + sq];
                    const double tau = (aqq - app) / (2.0 * apq);
                    t = tau >= 0.0 ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                   : -1.0 / (-tau + sqrt(1.0 + tau * tau));
                    c = 1.0 / sqrt(1.0 + t * t);
                    s = t * c;
                }
                rc[pr] = c;
                rs[pr] = s;
                rt[pr] = t;
                ra[pr] = apq;
            }
            __syncthreads();
            // M' = J^T M J over 2x2 blocks (P, Q); write in the next slot order.
            for (int64_t e = gtid; e < half * half; e += gstride) {
                const int64_t P = e / half, Q = e % half;
                const int64_t r0 = 2 * P, c0 = 2 * Q;
                const double2 top = *reinterpret_cast<const double2*>(M + r0 * W2 + c0);
                const double2 bot = *reinterpret_cast<const double2*>(M + (r0 + 1) * W2 + c0);
                double o00, o01, o10, o11;
                if (P == Q) {
                    if (!(fabs(ra[P]) <= skip)) {
                        const double tt = rt[P], apq = ra[P];
                        o00 = top.x - tt * apq;
                        o11 = bot.y + tt * apq;
                        o01 = 0.0;
                        o10 = 0.0;
                    } else {
                        o00 = top.x; o01 = top.y; o10 = bot.x; o11 = bot.y;
                    }
                } else {
                    const double cq = rc[Q], sq = rs[Q], cp = rc[P], spp = rs[P];
                    // column rotation (right multiply by J_Q)
                    const double a0 = cq * top.x - sq * top.y, a1 = sq * top.x + cq * top.y;
                    const double b0 = cq * bot.x - sq * bot.y, b1 = sq * bot.x + cq * bot.y;
                    // row rotation (left multiply by J_P^T)
                    o00 = cp * a0 - spp * b0;
                    o01 = cp * a1 - spp * b1;
                    o10 = spp * a0 + cp * b0;
                    o11 = spp * a1 + cp * b1;
                }
                const int64_t nr0 = next_slot(r0, W2), nr1 = next_slot(r0 + 1, W2);
                const int64_t nc0 = next_slot(c0, W2), nc1 = next_slot(c0 + 1, W2);
                Mn[nr0 * W2 + nc0] = o00;
                Mn[nr0 * W2 + nc1] = o01;
                Mn[nr1 * W2 + nc0] = o10;
                Mn[nr1 * W2 + nc1] = o11;
            }
            // V' = V J (columns in slot order)
            for (int64_t e = gtid; e < st.nv * half; e += gstride) {
                const int64_t i = e / half, Q = e % half;
                const double2 x = *reinterpret_cast<const double2*>(V + i * W2 + 2 * Q);
                const double c = rc[Q], s = rs[Q];
                Vn[i * W2 + next_slot(2 * Q, W2)] = c * x.x - s * x.y;
                Vn[i * W2 + next_slot(2 * Q + 1, W2)] = s * x.x + c * x.y;
            }
            cur ^= 1;
            grid_barrier(st.bar, gridDim.x);
        }
        ++sweeps;
        double o2 = 0.0;
        const double* M = st.Mb[cur];
        for (int64_t e = gtid; e < W2 * W2; e += gstride) {
            if (e / W2 != e % W2) {
                double x = M[e];
                o2 += x * x;
            }
        }
        off = sqrt(grid_sum(o2, st.partial, st.bar));
        converged = off <= threshold;
    }
    if (gtid == 0) {
        st.info[0] = converged ? 1 : 0;
        st.info[1] = sweeps;
        st.info[2] = cur;
        st.off_out[0] = off;
    }
}

__global__ void k_pad_copy(int64_t n, int64_t W2, const double* __restrict__ src, int64_t lds,
                           double* __restrict__ dst, int64_t rows) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * W2) return;
    int64_t i = e / W2, j = e % W2;
    dst[e] = (i < n && j < n) ? src[i * lds + j] : 0.0;
}

// Copy back from whichever ping-pong buffer holds the result (info[2]).
__global__ void k_unpad_copy(int64_t n, int64_t W2, const double* b0, const double* b1,
                             const int32_t* info, double* __restrict__ dst, int64_t ldd,
                             int64_t rows) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * n) return;
    int64_t i = e / n, j = e % n;
    const double* src = info[2] ? b1 : b0;
    dst[i * ldd + j] = src[i * W2 + j];
}

// ---------------------------------------------------------------------------
// eig_select
__global__ void k_eig_order(int64_t w, const double* __restrict__ M, int64_t ldm, int64_t k,
                            int32_t* __restrict__ order, double* __restrict__ evals) {
    for (int64_t i = threadIdx.x; i < w; i += blockDim.x) {
        const double di = M[i * ldm + i];
        int64_t rank = 0;
        for (int64_t j = 0; j < w; ++j) {
            const double dj = M[j * ldm + j];
            rank += (dj > di) || (dj == di && j < i);
        }
        if (rank < k) {
            order[rank] = (int32_t)i;
            evals[rank] = di;
        }
    }
}

__global__ void k_eig_gather(int64_t w, int64_t k, const int32_t* __restrict__ order,
                             const double* __restrict__ V, int64_t ldv, double* __restrict__ E,
                             int64_t lde) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= w * k) return;
    int64_t i = e / k, r = e % k;
    E[i * lde + r] = V[i * ldv + order[r]];
}


// ---------------------------------------------------------------------------
// Cholesky with deflation + in-place triangular inverse, one CTA, p <= kFastP.
// The packed upper triangle (row i holds columns i..p-1) lives in shared
// memory (201 KB at p = 224). Every step is spread over all threads:
//   factor, column j: uniform pivot test (factor.py:105 analogue) on the
//     Schur diagonal; scale row j (a deficient column gets R row j = e_j and
//     eliminates nothing); rank-1 update of the trailing triangle;
//   invert, row i from the bottom (T = R^{-1} in place): row i of T is the
//     accumulated row i over R_ii; column i of R (rows k < i) is staged, then
//     rows k < i take the rank-1 update X[k][c] -= R[k][i] T[i][c], c >= i.
// R with deficient rows e_j is invertible and (R^{-1})_SS = (R_SS)^{-1} on
// the kept set S, so zeroing the deficient rows and columns of the full
// inverse gives the restricted inverse.
#ifdef RSVD_CHOL_TRACE
__device__ long long g_chol_trace[64];
#define CHOL_T(i) do { if (threadIdx.x == 0 && (i) < 64) g_chol_trace[i] = clock64(); } while (0)
// phase accumulators (thread 0): CHOL_P0() at kernel start, CHOL_P(i) adds the cycles since the last mark to slot i
#define CHOL_P0() long long chol_pm = clock64(); do { if (threadIdx.x == 0) for (int q_ = 8; q_ < 16; ++q_) g_chol_trace[q_] = 0; } while (0)
#define CHOL_P(i) do { const long long now_ = clock64(); if (threadIdx.x == 0) g_chol_trace[i] += now_ - chol_pm; chol_pm = now_; } while (0)
#else
#define CHOL_T(i) do { } while (0)
#define CHOL_P0() do { } while (0)
#define CHOL_P(i) do { } while (0)
#endif
constexpr int kSwThreadsMax = 512;
constexpr int kChNB = 16;  // block-row height of the blocked factorization

__global__ void __launch_bounds__(kSwThreadsMax)
k_chol_sweep(int p, const double* __restrict__ G, int64_t ldg, const double* __restrict__ ref2, double tau2,
             double* __restrict__ T, int64_t ldt, int32_t* __restrict__ mask, int32_t* __restrict__ ndef,
             int32_t* __restrict__ running, const int32_t* __restrict__ active, const int32_t* __restrict__ pred,
             int blocked, int inv_blocked) {
    if (pred && *pred == 0) return;
    extern __shared__ double S[];
    __shared__ int s_row[kFastP];  // S[s_row[i] + j] = element (i, j), j >= i
    __shared__ double s_ref[kFastP];
    __shared__ double s_vec[kFastP];   // staged row j (factor) / column i (invert)
    __shared__ double s_vec2[kFastP];  // staged row i (invert)
    __shared__ int s_msk[kFastP];      // 0 kept, 1 deficient, 2 inactive
    __shared__ double s_piv[2];        // factor: inv (0 if deficient), rjj; invert: rinv
    __shared__ int s_def, s_count;
    const int nt = blockDim.x, tid = threadIdx.x, tx = tid & 31, ty = tid >> 5, ny = nt >> 5;
    for (int i = tid; i < p; i += nt) {
        s_row[i] = i * p - (i * (i - 1)) / 2 - i;
        s_ref[i] = ref2 ? ref2[i] : G[(int64_t)i * ldg + i];
        s_msk[i] = (active && active[i] == 0) ? 2 : 0;
    }
    if (tid == 0) s_count = 0;
    __syncthreads();
    for (int i = ty; i < p; i += ny)
        for (int j = i + tx; j < p; j += 32) S[s_row[i] + j] = G[(int64_t)i * ldg + j];
    __syncthreads();
    CHOL_T(0);
    // Right-looking, blocked by kChNB columns: a column step updates only the
    // rows of its block row (all their columns); after the block row is done,
    // the trailing triangle takes one rank-kChNB update (each element read and
    // written once per block instead of once per column). Thread mapping of
    // that update: one warp per (4-row group, 64-column chunk), lanes on
    // columns c and c + 32, the 4 rows' R entries read by broadcast.
    const int nb = blocked ? kChNB : p;
    for (int k0 = 0; k0 < p; k0 += nb) {
        const int k1 = min(k0 + nb, p);
        for (int j = k0; j < k1; ++j) {
            const int rj = s_row[j];
            // A: stage row j (unscaled); thread 0 takes the pivot decision
            for (int c = j + tid; c < p; c += nt) s_vec[c] = S[rj + c];
            if (tid == 0) {
                const double d = S[rj + j];
                const int inactive = s_msk[j] == 2;
                const bool def = inactive || !(d > tau2 * s_ref[j]) || !(d > 0.0);
                const double rjj = def ? 1.0 : sqrt(d);
                s_piv[0] = def ? 0.0 : 1.0 / rjj;
                s_piv[1] = rjj;
                s_def = def;
                if (def && !inactive) {
                    s_msk[j] = 1;
                    ++s_count;
                }
            }
            __syncthreads();
            // B: scale row j; rank-1 update of the block row's remaining rows
            const double inv = s_piv[0];
            if (ty == 0)
                for (int c = j + tx; c < p; c += 32) S[rj + c] = (c == j) ? s_piv[1] : s_vec[c] * inv;
            if (!s_def) {
                for (int i = j + 1 + ty; i < k1; i += ny) {
                    const double ui = s_vec[i] * inv;
                    double* row = S + s_row[i];
                    for (int c = i + tx; c < p; c += 32) row[c] = fma(-ui, s_vec[c] * inv, row[c]);
                }
            }
            __syncthreads();
        }
        if (k1 >= p) break;
        // C: trailing update S[i][c] -= sum_{j in [k0,k1)} R[j][i] R[j][c], k1 <= i <= c
        const int mt = p - k1;
        const int ngr = (mt + 3) / 4, nch = (mt + 63) / 64;
        for (int item = ty; item < ngr * nch; item += ny) {
            const int g = item / nch, ch = item % nch;
            const int i0 = k1 + 4 * g;
            const int cbase = k1 + 64 * ch;
            if (cbase + 63 < i0) continue;  // chunk entirely below the diagonal (warp-uniform)
            const int c0 = cbase + tx, c1 = c0 + 32;
            double acc[4][2];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a][0] = acc[a][1] = 0.0;
            for (int j = k0; j < k1; ++j) {
                const double* rjp = S + s_row[j];
                const double b0 = c0 < p ? rjp[c0] : 0.0, b1 = c1 < p ? rjp[c1] : 0.0;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const double ra = i0 + a < p ? rjp[i0 + a] : 0.0;
                    acc[a][0] = fma(ra, b0, acc[a][0]);
                    acc[a][1] = fma(ra, b1, acc[a][1]);
                }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int i = i0 + a;
                if (i >= p) break;
                double* row = S + s_row[i];
                if (c0 >= i && c0 < p) row[c0] -= acc[a][0];
                if (c1 >= i && c1 < p) row[c1] -= acc[a][1];
            }
        }
        __syncthreads();
    }
    CHOL_T(1);
    // In-place inversion from the bottom. Blocked (inv_blocked): the rows of a
    // kChNB-row block are finalised one by one updating only the block's own
    // rows; then every row above takes the block's contribution in one pass
    //   X[k][c] = -sum_{i0 <= i <= c} R[k][i] T[i][c]   (c inside the block:
    //             the entry held R[k][c] and is replaced, as the column step does)
    //   X[k][c] -= sum_{i in block} R[k][i] T[i][c]     (c past the block)
    // with the block's R[k][i] staged in Rb first (the pass overwrites them).
    const int nbi = inv_blocked ? kChNB : p;
    double* Rb = S + (p * (p + 1)) / 2;  // [p][kChNB] (inv_blocked only)
    for (int i1 = p; i1 > 0; i1 -= nbi) {
        const int i0 = max(0, i1 - nbi);
        for (int i = i1 - 1; i >= i0; --i) {
            const int ri = s_row[i];
            // A: stage column i (block rows k < i) and row i of the accumulated inverse
            for (int k = i0 + tid; k < i; k += nt) s_vec[k] = S[s_row[k] + i];
            for (int c = i + tid; c < p; c += nt) s_vec2[c] = S[ri + c];
            __syncthreads();
            // B: row i of T = accumulated row / R_ii; block rows k < i: X[k][c] -= R[k][i] T[i][c]
            const double rinv = 1.0 / s_vec2[i];
            if (ty == 0)
                for (int c = i + tx; c < p; c += 32) S[ri + c] = (c == i) ? rinv : s_vec2[c] * rinv;
            for (int k = i0 + ty; k < i; k += ny) {
                const double rk = s_vec[k];
                double* row = S + s_row[k];
                for (int c = i + tx; c < p; c += 32) {
                    const double tic = (c == i) ? rinv : s_vec2[c] * rinv;
                    row[c] = (c == i) ? -rk * tic : fma(-rk, tic, row[c]);
                }
            }
            __syncthreads();
        }
        if (i0 == 0 || !inv_blocked) continue;
        const int nb = i1 - i0;
        for (int e = tid; e < i0 * kChNB; e += nt) {
            const int k = e / kChNB, ii = e % kChNB;
            Rb[e] = ii < nb ? S[s_row[k] + i0 + ii] : 0.0;
        }
        __syncthreads();
        const int ngr = (i0 + 3) / 4, nch = (p - i0 + 63) / 64;
        for (int item = ty; item < ngr * nch; item += ny) {
            const int g = item / nch, ch = item % nch;
            const int k0 = 4 * g;
            const int c0 = i0 + 64 * ch + tx, c1 = c0 + 32;
            double acc[4][2];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a][0] = acc[a][1] = 0.0;
            for (int ii = 0; ii < nb; ++ii) {
                const int i = i0 + ii;
                const double* ti = S + s_row[i];
                const double t0 = (c0 >= i && c0 < p) ? ti[c0] : 0.0;
                const double t1 = (c1 >= i && c1 < p) ? ti[c1] : 0.0;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const double rk = k0 + a < i0 ? Rb[(k0 + a) * kChNB + ii] : 0.0;
                    acc[a][0] = fma(rk, t0, acc[a][0]);
                    acc[a][1] = fma(rk, t1, acc[a][1]);
                }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int k = k0 + a;
                if (k >= i0) break;
                double* row = S + s_row[k];
                if (c0 < p) row[c0] = c0 < i1 ? -acc[a][0] : row[c0] - acc[a][0];
                if (c1 < p) row[c1] = c1 < i1 ? -acc[a][1] : row[c1] - acc[a][1];
            }
        }
        __syncthreads();
    }
    CHOL_T(2);
    for (int c = ty; c < p; c += ny)
        for (int a = tx; a < p; a += 32)
            T[(int64_t)c * ldt + a] = (a < c || s_msk[c] || s_msk[a]) ? 0.0 : S[s_row[c] + a];
    for (int j = tid; j < p; j += nt) mask[j] = s_msk[j] == 1 ? 1 : 0;
    if (tid == 0) {
        const int32_t base = running ? running[0] : 0;
        ndef[0] = s_count;
        ndef[1] = base;
        if (running) running[0] = base + s_count;
    }
    CHOL_T(3);
}

// k_chol_sweep's blocked arithmetic (bitwise equal: every matrix entry sees
// the same operations in the same order) with the per-column barriers taken
// out of the block rows. k_chol_sweep spends two block barriers per column in
// both phases (2 x 2 x p of them, ~1 us each: 330 us at p = 200). Here, per
// 16-column block:
//   factor: ONE WARP factors the 16 x 16 diagonal block with the column
//     entries in registers and shuffles (pivot test, sqrt, reciprocal and the
//     in-block rank-1 updates: no block barrier), and publishes the block's
//     R, the pivot reciprocals and the deficiency flags; then every column
//     right of the block runs the 16 elimination steps on its own 16 entries
//     in registers (thread per column, no communication); then the trailing
//     triangle takes the rank-16 update as before;
//   invert: the 16 x 16 block of R is staged once; every column c >= i0 then
//     runs the block's 16 back-substitution steps on its own entries in
//     registers (the steps of a column only read that column and the staged
//     block); then the rows above take the block's contribution as before.
// Three barriers per block instead of 32 + 2.
constexpr int kBk = 16;

__global__ void __launch_bounds__(256, 1)
k_chol_blk(int p, const double* __restrict__ G, int64_t ldg, const double* __restrict__ ref2, double tau2,
           double* __restrict__ T, int64_t ldt, int32_t* __restrict__ mask, int32_t* __restrict__ ndef,
           int32_t* __restrict__ running, const int32_t* __restrict__ active, const int32_t* __restrict__ pred) {
    if (pred && *pred == 0) return;
    extern __shared__ double S[];
    __shared__ int s_row[kFastP];  // S[s_row[i] + j] = element (i, j), j >= i
    __shared__ double s_ref[kFastP];
    __shared__ int s_msk[kFastP];  // 0 kept, 1 deficient, 2 inactive
    __shared__ double s_blk[kBk][kBk + 1];
    __shared__ double s_inv[kBk];
    __shared__ int s_dfl[kBk];
    __shared__ int s_count;
    const int nt = blockDim.x, tid = threadIdx.x, tx = tid & 31, ty = tid >> 5, ny = nt >> 5;
    for (int i = tid; i < p; i += nt) {
        s_row[i] = i * p - (i * (i - 1)) / 2 - i;
        s_ref[i] = ref2 ? ref2[i] : G[(int64_t)i * ldg + i];
        s_msk[i] = (active && active[i] == 0) ? 2 : 0;
    }
    if (tid == 0) s_count = 0;
    __syncthreads();
    for (int i = ty; i < p; i += ny)
        for (int j = i + tx; j < p; j += 32) S[s_row[i] + j] = G[(int64_t)i * ldg + j];
    __syncthreads();
    CHOL_T(0);
    CHOL_P0();
    for (int k0 = 0; k0 < p; k0 += kBk) {
        const int nb = min(kBk, p - k0), k1 = k0 + nb;
        if (ty == 0) {
            // D: lane l holds column k0 + l of the diagonal block (rows k0 .. k0 + l)
            const int l = tx;
            double x[kBk];
#pragma unroll
            for (int t = 0; t < kBk; ++t) x[t] = (l < nb && t <= l) ? S[s_row[k0 + t] + k0 + l] : 0.0;
            int cnt = 0;
#pragma unroll
            for (int j = 0; j < kBk; ++j) {
                if (j < nb) {  // warp-uniform
                    double rjj = 1.0, inv = 0.0;
                    int dfl = 0;
                    if (l == j) {
                        const double d = x[j];
                        const int inactive = s_msk[k0 + j] == 2;
                        const bool def = inactive || !(d > tau2 * s_ref[k0 + j]) || !(d > 0.0);
                        rjj = def ? 1.0 : sqrt(d);
                        inv = def ? 0.0 : 1.0 / rjj;
                        dfl = def;
                        if (def && !inactive) {
                            s_msk[k0 + j] = 1;
                            ++cnt;
                        }
                        s_inv[j] = inv;
                        s_dfl[j] = dfl;
                    }
                    inv = __shfl_sync(0xffffffffu, inv, j);
                    rjj = __shfl_sync(0xffffffffu, rjj, j);
                    dfl = __shfl_sync(0xffffffffu, dfl, j);
                    const double sv = x[j] * inv;  // scaled row j at this lane's column (lanes >= j)
                    x[j] = (l == j) ? rjj : sv;
#pragma unroll
                    for (int i = j + 1; i < kBk; ++i) {
                        const double ui = __shfl_sync(0xffffffffu, sv, i);  // R[j][k0 + i]
                        if (!dfl && i < nb && i <= l) x[i] = fma(-ui, sv, x[i]);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < kBk; ++t)
                if (l < nb && t <= l) {
                    S[s_row[k0 + t] + k0 + l] = x[t];
                    s_blk[t][l] = x[t];
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if (l == 0) s_count += cnt;
        }
        __syncthreads();
        CHOL_P(8);
        if (k1 >= p) break;
        // P: columns right of the block, the block's nb elimination steps in registers
        for (int c = k1 + tid; c < p; c += nt) {
            double x[kBk];
#pragma unroll
            for (int t = 0; t < kBk; ++t) x[t] = t < nb ? S[s_row[k0 + t] + c] : 0.0;
#pragma unroll
            for (int j = 0; j < kBk; ++j) {
                if (j < nb) {
                    const double sv = x[j] * s_inv[j];
                    x[j] = sv;
                    if (!s_dfl[j]) {
#pragma unroll
                        for (int i = j + 1; i < kBk; ++i)
                            if (i < nb) x[i] = fma(-s_blk[j][i], sv, x[i]);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < kBk; ++t)
                if (t < nb) S[s_row[k0 + t] + c] = x[t];
        }
        __syncthreads();
        CHOL_P(9);
        // C: trailing update S[i][c] -= sum_{j in [k0,k1)} R[j][i] R[j][c], k1 <= i <= c
        const int mt = p - k1;
        const int ngr = (mt + 3) / 4, nch = (mt + 63) / 64;
        for (int item = ty; item < ngr * nch; item += ny) {
            const int g = item / nch, ch = item % nch;
            const int i0 = k1 + 4 * g;
            const int cbase = k1 + 64 * ch;
            if (cbase + 63 < i0) continue;  // chunk entirely below the diagonal (warp-uniform)
            const int c0 = cbase + tx, c1 = c0 + 32;
            double acc[4][2];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a][0] = acc[a][1] = 0.0;
            for (int j = k0; j < k1; ++j) {
                const double* rjp = S + s_row[j];
                const double b0 = c0 < p ? rjp[c0] : 0.0, b1 = c1 < p ? rjp[c1] : 0.0;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const double ra = i0 + a < p ? rjp[i0 + a] : 0.0;
                    acc[a][0] = fma(ra, b0, acc[a][0]);
                    acc[a][1] = fma(ra, b1, acc[a][1]);
                }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int i = i0 + a;
                if (i >= p) break;
                double* row = S + s_row[i];
                if (c0 >= i && c0 < p) row[c0] -= acc[a][0];
                if (c1 >= i && c1 < p) row[c1] -= acc[a][1];
            }
        }
        __syncthreads();
        CHOL_P(10);
    }
    CHOL_T(1);
    // in-place inversion from the bottom, block by block
    double* Rb = S + (p * (p + 1)) / 2;  // [p][kBk]
    for (int i1 = p; i1 > 0; i1 -= kBk) {
        const int i0 = max(0, i1 - kBk), nb = i1 - i0;
        // the block's R (rows and columns i0 .. i1 - 1) and its pivots' reciprocals
        for (int e = tid; e < kBk * kBk; e += nt) {
            const int k = e / kBk, i = e % kBk;
            if (k <= i && i < nb) {
                const double v = S[s_row[i0 + k] + i0 + i];
                s_blk[k][i] = v;
                if (k == i) s_inv[i] = 1.0 / v;
            }
        }
        __syncthreads();
        for (int c = i0 + tid; c < p; c += nt) {
            const int tc = c - i0;  // in-block column when tc < nb
            double x[kBk];
#pragma unroll
            for (int t = 0; t < kBk; ++t) x[t] = (t < nb && t <= tc) ? S[s_row[i0 + t] + c] : 0.0;
#pragma unroll
            for (int t = kBk - 1; t >= 0; --t) {
                if (t < nb && t <= tc) {
                    const double rinv = s_inv[t];
                    const double tic = (t == tc) ? rinv : x[t] * rinv;
                    x[t] = tic;
#pragma unroll
                    for (int k = 0; k < t; ++k) {
                        const double rk = s_blk[k][t];
                        x[k] = (t == tc) ? -rk * tic : fma(-rk, tic, x[k]);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < kBk; ++t)
                if (t < nb && t <= tc) S[s_row[i0 + t] + c] = x[t];
        }
        __syncthreads();
        CHOL_P(11);
        if (i0 == 0) break;
        for (int e = tid; e < i0 * kBk; e += nt) {
            const int k = e / kBk, ii = e % kBk;
            Rb[e] = ii < nb ? S[s_row[k] + i0 + ii] : 0.0;
        }
        __syncthreads();
        const int ngr = (i0 + 3) / 4, nch = (p - i0 + 63) / 64;
        for (int item = ty; item < ngr * nch; item += ny) {
            const int g = item / nch, ch = item % nch;
            const int k0 = 4 * g;
            const int c0 = i0 + 64 * ch + tx, c1 = c0 + 32;
            double acc[4][2];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a][0] = acc[a][1] = 0.0;
            for (int ii = 0; ii < nb; ++ii) {
                const int i = i0 + ii;
                const double* ti = S + s_row[i];
                const double t0 = (c0 >= i && c0 < p) ? ti[c0] : 0.0;
                const double t1 = (c1 >= i && c1 < p) ? ti[c1] : 0.0;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const double rk = k0 + a < i0 ? Rb[(k0 + a) * kBk + ii] : 0.0;
                    acc[a][0] = fma(rk, t0, acc[a][0]);
                    acc[a][1] = fma(rk, t1, acc[a][1]);
                }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int k = k0 + a;
                if (k >= i0) break;
                double* row = S + s_row[k];
                if (c0 < p) row[c0] = c0 < i1 ? -acc[a][0] : row[c0] - acc[a][0];
                if (c1 < p) row[c1] = c1 < i1 ? -acc[a][1] : row[c1] - acc[a][1];
            }
        }
        __syncthreads();
        CHOL_P(12);
    }
    CHOL_T(2);
    for (int c = ty; c < p; c += ny)
        for (int a = tx; a < p; a += 32)
            T[(int64_t)c * ldt + a] = (a < c || s_msk[c] || s_msk[a]) ? 0.0 : S[s_row[c] + a];
    for (int j = tid; j < p; j += nt) mask[j] = s_msk[j] == 1 ? 1 : 0;
    if (tid == 0) {
        const int32_t base = running ? running[0] : 0;
        ndef[0] = s_count;
        ndef[1] = base;
        if (running) running[0] = base + s_count;
    }
    CHOL_T(3);
}

// p <= 64: thread t holds column t of the Schur complement / R in registers.
// Per column j: thread j
// takes the pivot decision (rsqrt), the scaled row j goes through shared
// memory, and each thread updates its own column (2 barriers of 64 threads
// per step; entries below a column's diagonal are never read, so the update
// runs unpredicated). The inverse is a column sweep with x in registers, R
// read by broadcast and the pivots' reciprocals kept from the factorization.
// (Measured at p = 50: ~37k cycles factor + ~24k inverse; a one-warp variant
// without block barriers, k_chol_warp, is slower: LDS latency is not hidden.)
constexpr int kRegP = 64;

#ifndef RSVD_CHOL_UNROLL
#define RSVD_CHOL_UNROLL 1
#endif
constexpr int kChUnroll = RSVD_CHOL_UNROLL;
// The steps are a real loop and every register index is static because the
// register window rotates by one each step (r[0] is always the current pivot
// row's entry). (A fully unrolled variant, bitwise equal, was 64 KB of
// straight-line code fetched cold from HBM on every call inside a
// factorization -- the chain's 2 GB stream evicts it from L2: 83 us cold vs
// 34 us warm at p = 50 -- and was removed; this one is ~3 KB.)
__global__ void __launch_bounds__(kRegP)
k_chol_reg64c(int p, const double* __restrict__ G, int64_t ldg, const double* __restrict__ ref2, double tau2,
              double* __restrict__ T, int64_t ldt, int32_t* __restrict__ mask, int32_t* __restrict__ ndef,
              int32_t* __restrict__ running, const int32_t* __restrict__ active, const int32_t* __restrict__ pred) {
    if (pred && *pred == 0) return;
    __shared__ double Rs[kRegP][kRegP + 1];  // R(i, c) = Rs[i][c]
    __shared__ double s_row[2 * kRegP];      // scaled row j (entries >= kRegP stay 0)
    __shared__ double s_piv[2];
    __shared__ double s_rinv[kRegP];
    __shared__ int s_msk[kRegP];
    __shared__ int s_def, s_count;
    const int t = threadIdx.x;
    const bool mine = t < p;
    double r[kRegP];  // r[i] = element (j + i, t) at step j
#pragma unroll
    for (int i = 0; i < kRegP; ++i) r[i] = (mine && i <= t) ? G[(int64_t)i * ldg + t] : 0.0;
    const double myref = mine ? (ref2 ? ref2[t] : G[(int64_t)t * ldg + t]) : 0.0;
    const int myinact = mine ? (active && active[t] == 0) : 1;
    s_msk[t] = myinact && mine ? 2 : 0;
    s_row[kRegP + t] = 0.0;
    if (t == 0) s_count = 0;
    __syncthreads();
#pragma unroll (kChUnroll)
    for (int j = 0; j < p; ++j) {
        if (t == j) {
            const double d = r[0];
            const bool def = myinact || !(d > tau2 * myref) || !(d > 0.0);
            const double inv = def ? 0.0 : rsqrt(d);
            s_piv[0] = inv;
            s_piv[1] = def ? 1.0 : d * inv;
            s_rinv[j] = def ? 1.0 : inv;
            s_def = def;
            if (def && !myinact) {
                s_msk[j] = 1;
                ++s_count;
            }
        }
        __syncthreads();
        const double inv = s_piv[0];
        if (t == j) r[0] = s_piv[1];
        else if (t > j) r[0] *= inv;
        s_row[t] = r[0];  // R(j, t) for t > j
        Rs[j][t] = (mine && j <= t) ? r[0] : 0.0;
        const bool def = s_def;
        __syncthreads();
        if (!def) {
            const double rj = r[0];
#pragma unroll
            for (int i = 1; i < kRegP; ++i) r[i] = fma(-s_row[j + i], rj, r[i]);
        }
#pragma unroll
        for (int i = 0; i + 1 < kRegP; ++i) r[i] = r[i + 1];
        r[kRegP - 1] = 0.0;
    }
    for (int j = p; j < kRegP; ++j) Rs[j][t] = 0.0;
    __syncthreads();
    // column t of T: R x = e_t from the bottom; y[m] = x[i - m] at step i
    double y[kRegP];
#pragma unroll
    for (int m = 0; m < kRegP; ++m) y[m] = (p - 1 - m == t) ? 1.0 : 0.0;
    const bool zc = mine && s_msk[t] != 0;
#pragma unroll (kChUnroll)
    for (int i = p - 1; i >= 0; --i) {
        const double xi = y[0] * s_rinv[i];
        if (mine) T[(int64_t)i * ldt + t] = (i > t || zc || s_msk[i]) ? 0.0 : xi;
#pragma unroll
        for (int m = 1; m < kRegP; ++m)
            if (i - m >= 0) y[m] = fma(-Rs[i - m][i], xi, y[m]);
#pragma unroll
        for (int m = 0; m + 1 < kRegP; ++m) y[m] = y[m + 1];
        y[kRegP - 1] = 0.0;
    }
    if (mine) mask[t] = s_msk[t] == 1 ? 1 : 0;
    if (t == 0) {
        const int32_t base = running ? running[0] : 0;
        ndef[0] = s_count;
        ndef[1] = base;
        if (running) running[0] = base + s_count;
    }
}

// k_chol_reg64c with two threads per column (128 threads): thread (c, h)
// holds rows 32h .. 32h+31 of column c, and only the half that contains the
// current pivot row rotates its window, so each thread shifts and updates at
// most 32 registers per step. Every matrix entry still sees the same
// operations in the same order (bitwise equal to k_chol_reg64c); the
// inversion needs one extra barrier per row to hand x_i to the other half.
constexpr int kRegH = 32;

__global__ void __launch_bounds__(2 * kRegP)
k_chol_reg64h(int p, const double* __restrict__ G, int64_t ldg, const double* __restrict__ ref2, double tau2,
              double* __restrict__ T, int64_t ldt, int32_t* __restrict__ mask, int32_t* __restrict__ ndef,
              int32_t* __restrict__ running, const int32_t* __restrict__ active, const int32_t* __restrict__ pred) {
    if (pred && *pred == 0) return;
    __shared__ double Rs[kRegP][kRegP + 1];
    __shared__ double s_row[2 * kRegP];
    __shared__ double s_x[kRegP];
    __shared__ double s_piv[2];
    __shared__ double s_rinv[kRegP];
    __shared__ int s_msk[kRegP];
    __shared__ int s_def, s_count;
    const int c = threadIdx.x & (kRegP - 1), h = threadIdx.x >> 6;
    const bool mine = c < p;
    const int rbase = kRegH * h;  // first row of this half
    double r[kRegH];              // r[i] = element (row_lo + i, c); row_lo = rbase, or j while rotating
#pragma unroll
    for (int i = 0; i < kRegH; ++i) {
        const int row = rbase + i;
        r[i] = (mine && row <= c) ? G[(int64_t)row * ldg + c] : 0.0;
    }
    const double myref = mine ? (ref2 ? ref2[c] : G[(int64_t)c * ldg + c]) : 0.0;
    const int myinact = mine ? (active && active[c] == 0) : 1;
    if (h == 0) {
        s_msk[c] = myinact && mine ? 2 : 0;
        s_row[kRegP + c] = 0.0;
    }
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
#pragma unroll 1
    for (int j = 0; j < p; ++j) {
        const int hj = j >> 5;
        const bool rot = h == hj;  // this half holds row j (its r[0])
        if (rot && c == j) {
            const double d = r[0];
            const bool def = myinact || !(d > tau2 * myref) || !(d > 0.0);
            const double inv = def ? 0.0 : rsqrt(d);
            s_piv[0] = inv;
            s_piv[1] = def ? 1.0 : d * inv;
            s_rinv[j] = def ? 1.0 : inv;
            s_def = def;
            if (def && !myinact) {
                s_msk[j] = 1;
                ++s_count;
            }
        }
        __syncthreads();
        if (rot) {
            const double inv = s_piv[0];
            if (c == j) r[0] = s_piv[1];
            else if (c > j) r[0] *= inv;
            s_row[c] = r[0];  // R(j, c) for c > j
            Rs[j][c] = (mine && j <= c) ? r[0] : 0.0;
        }
        const bool def = s_def;
        __syncthreads();
        if (!def) {
            const double rj = s_row[c];
            if (rot) {
#pragma unroll
                for (int i = 1; i < kRegH; ++i) r[i] = fma(-s_row[j + i], rj, r[i]);
            } else if (h > hj) {
#pragma unroll
                for (int i = 0; i < kRegH; ++i) r[i] = fma(-s_row[rbase + i], rj, r[i]);
            }
        }
        if (rot) {
#pragma unroll
            for (int i = 0; i + 1 < kRegH; ++i) r[i] = r[i + 1];
            r[kRegH - 1] = 0.0;
        }
    }
    if (h == 0)
        for (int j = p; j < kRegP; ++j) Rs[j][c] = 0.0;
    __syncthreads();
    // inversion: column c of T, R x = e_c from the bottom. Half h keeps
    // y[m] = x[top_h - m], top_h = min(i, 32h + 31) (rotating while i is in it)
    double y[kRegH];
    const int top0 = min(p - 1, rbase + kRegH - 1);
#pragma unroll
    for (int m = 0; m < kRegH; ++m) y[m] = (top0 - m == c && top0 - m >= rbase) ? 1.0 : 0.0;
    const bool zc = mine && s_msk[c] != 0;
#pragma unroll 1
    for (int i = p - 1; i >= 0; --i) {
        const int hi = i >> 5;
        if (h == hi) {
            const double xi = y[0] * s_rinv[i];
            s_x[c] = xi;
            if (mine) T[(int64_t)i * ldt + c] = (i > c || zc || s_msk[i]) ? 0.0 : xi;
        }
        __syncthreads();
        const double xi = s_x[c];
        if (h == hi) {
#pragma unroll
            for (int m = 1; m < kRegH; ++m)
                if (i - m >= rbase) y[m] = fma(-Rs[i - m][i], xi, y[m]);
#pragma unroll
            for (int m = 0; m + 1 < kRegH; ++m) y[m] = y[m + 1];
            y[kRegH - 1] = 0.0;
        } else if (h < hi) {
#pragma unroll
            for (int m = 0; m < kRegH; ++m) y[m] = fma(-Rs[rbase + kRegH - 1 - m][i], xi, y[m]);
        }
        __syncthreads();  // s_x is rewritten next row
    }
    if (h == 0 && mine) mask[c] = s_msk[c] == 1 ? 1 : 0;
    if (threadIdx.x == 0) {
        const int32_t base = running ? running[0] : 0;
        ndef[0] = s_count;
        ndef[1] = base;
        if (running) running[0] = base + s_count;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// public wrappers (called from api.cu)

int64_t chol_deflate_ws_bytes(int64_t p) { return (p * (p + 1) / 2) * (int64_t)sizeof(double); }

int chol_deflate(int64_t p, const double* G, int64_t ldg, const double* ref2, double tau2, double* T,
                 int64_t ldt, int32_t* mask, int32_t* ndef, int32_t* running, const int32_t* active, void* ws,
                 int64_t ws_bytes, const int32_t* pred, cudaStream_t st) {
    if (p == 0) return RSVD_OK;
    static const bool force_sweep = getenv("RSVD_CHOL_SWEEP") != nullptr;  // A/B experiments
    if (p <= kRegP && !force_sweep) {
        if (getenv("RSVD_CHOL_REG_ONE") == nullptr)  // default: two threads per column
            k_chol_reg64h<<<1, 2 * kRegP, 0, st>>>((int)p, G, ldg, ref2, tau2, T, ldt, mask, ndef, running, active,
                                                   pred);
        else
            k_chol_reg64c<<<1, kRegP, 0, st>>>((int)p, G, ldg, ref2, tau2, T, ldt, mask, ndef, running, active,
                                               pred);
        RSVD_CHECK_LAUNCH();
        return RSVD_OK;
    }
    if (p <= kFastP) {
        const size_t tri = (size_t)(p * (p + 1) / 2) * sizeof(double);
        const int blocked = getenv("RSVD_CHOL_UNBLOCKED") == nullptr;  // A/B switch
        // blocked inversion needs a p x kChNB staging block next to the triangle
        const size_t smb = tri + (size_t)p * kChNB * sizeof(double);
        const int inv_blocked = blocked && smb <= 200 * 1024;
        const size_t sm = inv_blocked ? smb : tri;
        if (sm > 48 * 1024)
            RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_chol_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        const int nt = p <= 64 ? 128 : (p <= 128 ? 256 : kSwThreadsMax);
        // default: the barrier-light blocked kernel (bitwise equal to the blocked sweep;
        // RSVD_CHOL_SWEEP_OLD=1: k_chol_sweep, for A/B measurement)
        const bool old_sweep = getenv("RSVD_CHOL_SWEEP_OLD") != nullptr;
        if (inv_blocked && !old_sweep) {
            static PerDevice<bool> attr_dev;
            bool& attr = attr_dev.get();
            if (!attr) {
                RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_chol_blk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     200 * 1024));
                attr = true;
            }
            // 256 threads: one per column in the register phases (p <= 224), and 252
            // registers each (at 512 threads the unrolled block steps spill)
            k_chol_blk<<<1, nt > 256 ? 256 : nt, sm, st>>>((int)p, G, ldg, ref2, tau2, T, ldt, mask, ndef, running,
                                                          active, pred);
            RSVD_CHECK_LAUNCH();
            return RSVD_OK;
        }
        k_chol_sweep<<<1, nt, sm, st>>>((int)p, G, ldg, ref2, tau2, T, ldt, mask, ndef, running, active, pred,
                                         blocked, inv_blocked);
        RSVD_CHECK_LAUNCH();
        return RSVD_OK;
    }
    const int64_t rbytes = chol_deflate_ws_bytes(p);
    const int64_t tbytes = p * p * (int64_t)sizeof(double);
    const int64_t cap = 200 * 1024;
    int use_smem = rbytes <= cap;
    int t_in_smem = use_smem && rbytes + tbytes <= cap;
    if (!use_smem) RSVD_REQUIRE(ws && ws_bytes >= rbytes, "chol_deflate: workspace too small");
    size_t sm = (size_t)((use_smem ? rbytes : 0) + (t_in_smem ? tbytes : 0));
    if (sm > 48 * 1024)
        RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_chol_deflate, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sm));
    k_chol_deflate<<<1, kCholThreads, sm, st>>>(p, G, ldg, ref2, tau2, T, ldt, mask, ndef, running, active,
                                                (double*)ws, use_smem, t_in_smem, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

static int64_t jac_W2(int64_t n) { return n + (n & 1); }

int64_t jacobi_ws_bytes(int64_t n) {
    int64_t W2 = jac_W2(n);
    return (2 * W2 * W2 + 2 * n * W2 + 1024) * (int64_t)sizeof(double) + 64;
}

int jacobi_sweeps(int64_t n, double* M, int64_t ldm, double* V, int64_t ldv, double tol,
                  int max_sweeps, int32_t* info, double* off_out, void* ws, int64_t ws_bytes,
                  cudaStream_t st) {
    RSVD_REQUIRE(n >= 1, "jacobi: n must be >= 1");
    RSVD_REQUIRE(ws_bytes >= jacobi_ws_bytes(n), "jacobi: workspace too small");
    const int64_t W2 = jac_W2(n);
    double* base = (double*)ws;
    JacobiState s;
    s.n = n;
    s.W2 = W2;
    s.Mb[0] = base;
    s.Mb[1] = base + W2 * W2;
    s.Vb[0] = base + 2 * W2 * W2;
    s.Vb[1] = s.Vb[0] + n * W2;
    s.nv = n;
    s.partial = s.Vb[1] + n * W2;                // 1024 doubles (>= grid)
    s.bar = (unsigned int*)(s.partial + 1010);
    s.tol = tol;
    s.max_sweeps = max_sweeps;
    s.info = info;
    s.off_out = off_out;
    RSVD_CHECK_CUDA(cudaMemsetAsync(s.bar, 0, 2 * sizeof(unsigned int), st));
    unsigned nb = (unsigned)cdiv(W2 * W2, 256);
    k_pad_copy<<<nb, 256, 0, st>>>(n, W2, M, ldm, s.Mb[0], W2);
    RSVD_CHECK_LAUNCH();
    nb = (unsigned)cdiv(n * W2, 256);
    k_pad_copy<<<nb, 256, 0, st>>>(n, W2, V, ldv, s.Vb[0], n);
    RSVD_CHECK_LAUNCH();

    const int64_t half = W2 / 2;
    size_t smem = (size_t)(4 * half) * sizeof(double);
    RSVD_REQUIRE(smem <= 200 * 1024, "jacobi: n too large (%lld)", (long long)n);
    if (smem > 48 * 1024)
        RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
    int per_sm = 0;
    RSVD_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi, kJacThreads, smem));
    RSVD_REQUIRE(per_sm >= 1, "jacobi: kernel cannot be resident");
    int64_t want = cdiv(half * half + n * half, (int64_t)kJacThreads * 2);
    int64_t maxb = (int64_t)sm_count();
    if (want > maxb) want = maxb;
    if (want < 1) want = 1;
    unsigned grid = (unsigned)want;
    void* args[] = {&s};
    RSVD_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)k_jacobi, dim3(grid), dim3(kJacThreads),
                                                args, smem, st));
    nb = (unsigned)cdiv(n * n, 256);
    k_unpad_copy<<<nb, 256, 0, st>>>(n, W2, s.Mb[0], s.Mb[1], info, M, ldm, n);
    RSVD_CHECK_LAUNCH();
    k_unpad_copy<<<nb, 256, 0, st>>>(n, W2, s.Vb[0], s.Vb[1], info, V, ldv, n);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int eig_select(int64_t w, const double* M, int64_t ldm, const double* V, int64_t ldv, int64_t k,
               double* evals, double* evecs, int64_t lde, void* order_ws, cudaStream_t st) {
    RSVD_REQUIRE(k >= 0 && k <= w, "eig_select: k out of range");
    if (k == 0) return RSVD_OK;
    int32_t* order = (int32_t*)order_ws;
    k_eig_order<<<1, 1024, 0, st>>>(w, M, ldm, k, order, evals);
    RSVD_CHECK_LAUNCH();
    unsigned nb = (unsigned)cdiv(w * k, 256);
    k_eig_gather<<<nb, 256, 0, st>>>(w, k, order, V, ldv, evecs, lde);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace rsvd

#ifdef RSVD_CHOL_TRACE
extern "C" int rsvd_debug_chol_trace(long long* out) {
    return (int)cudaMemcpyFromSymbol(out, rsvd::g_chol_trace, sizeof(rsvd::g_chol_trace));
}
#endif
