// Top-k symmetric eigensolver for the Rayleigh-Ritz matrix M = Q^T A A^T Q
// (w x w, FP64), replacing the reference's full cyclic Jacobi
// (symmetric_eig, factor.py:132-166 -> _kernels.pyx:127-192) on the hot
// path. post_process only consumes the top k eigenpairs (rsvd.py:217-220),
// so this follows LAPACK's dsyevx structure:
//   1. Householder tridiagonalisation M = H T H^T: one cooperative kernel,
//      two grid barriers per column (matvec, then rank-2 update);
//   2. top-k eigenvalues of T by Sturm-count multisection (one warp per
//      eigenvalue, 32 shifts per step), to full FP64 accuracy;
//   3. eigenvectors of T by inverse iteration on a pivoted tridiagonal LU,
//      vectors of eigenvalue clusters (gap < 1e-5 ||T||_1) re-orthogonalised
//      in order (dstein's scheme), one warp per cluster;
//   4. back-transformation x <- H_0 ... H_{w-3} x, one warp per vector.
// Eigenvalues are returned descending; eigenvector signs are arbitrary (the
// caller canonicalises Z's signs, rsvd.py:192-197).
#include <cooperative_groups.h>

#include "common.cuh"

namespace rsvd {

namespace {

constexpr int kTriThreads = 512;

struct TriState {
    int64_t w;
    double* A;      // w x w work copy (row-major, ld = w), symmetric
    double* d;      // w
    double* e;      // w (e[i] couples i, i+1)
    double* Uh;     // w x w, row j = Householder vector of step j
    double* beta;   // w
    double* p;      // w scratch
    double* p2;     // w scratch (second p buffer of the one-barrier kernel)
    double* partial;
    unsigned int* bar;
};

__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    return s;
}

__global__ void __launch_bounds__(kTriThreads) k_tridiag(TriState s) {
    extern __shared__ double sh[];
    const int64_t w = s.w;
    double* u = sh;       // w
    double* q = sh + w;   // w
    __shared__ double red[kTriThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + tid) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = 0; j + 2 < w; ++j) {
        const int64_t m = w - j - 1;
        const double* rowj = s.A + j * w + (j + 1);
        double ss = 0.0, tail = 0.0;
        for (int64_t i = tid; i < m; i += blockDim.x) {
            const double x = rowj[i];
            u[i] = x;
            ss += x * x;
            if (i > 0) tail += x * x;
        }
        ss = block_sum(ss, red);
        tail = block_sum(tail, red);
        const double x0 = u[0];
        const bool skip = !(tail > 0.0);
        double alpha = x0, beta = 0.0;
        if (!skip) {
            const double nrm = sqrt(ss);
            alpha = x0 >= 0.0 ? -nrm : nrm;
            const double u0 = x0 - alpha;
            beta = 2.0 / (tail + u0 * u0);
            __syncthreads();
            if (tid == 0) u[0] = u0;
            __syncthreads();
        }
        if (blockIdx.x == 0) {
            if (tid == 0) {
                s.d[j] = s.A[j * w + j];
                s.e[j] = alpha;
                s.beta[j] = beta;
            }
            double* uh = s.Uh + j * w;
            for (int64_t i = tid; i < w; i += blockDim.x) uh[i] = (i > j && !skip) ? u[i - j - 1] : 0.0;
        }
        if (skip) continue;  // H_j = I: every CTA took the same decision
        // p = beta * A22 u  (warp per row)
        for (int64_t r = gwarp; r < m; r += nwarps) {
            const double* ar = s.A + (j + 1 + r) * w + (j + 1);
            double acc = 0.0;
            for (int64_t c = lane; c < m; c += 32) acc = fma(ar[c], u[c], acc);
            acc = warp_sum(acc);
            if (lane == 0) s.p[r] = beta * acc;
        }
        grid_barrier(s.bar, gridDim.x);
        double kk = 0.0;
        for (int64_t i = tid; i < m; i += blockDim.x) {
            const double pv = s.p[i];
            q[i] = pv;
            kk += u[i] * pv;
        }
        kk = 0.5 * beta * block_sum(kk, red);
        for (int64_t i = tid; i < m; i += blockDim.x) q[i] -= kk * u[i];
        __syncthreads();
        // A22 -= u q^T + q u^T
        for (int64_t r = gwarp; r < m; r += nwarps) {
            double* ar = s.A + (j + 1 + r) * w + (j + 1);
            const double ur = u[r], qr = q[r];
            for (int64_t c = lane; c < m; c += 32) ar[c] -= ur * q[c] + qr * u[c];
        }
        grid_barrier(s.bar, gridDim.x);
    }
    if (blockIdx.x == 0 && tid == 0) {
        if (w >= 2) {
            s.d[w - 2] = s.A[(w - 2) * w + (w - 2)];
            s.e[w - 2] = s.A[(w - 2) * w + (w - 1)];
            s.beta[w - 2] = 0.0;
        }
        s.d[w - 1] = s.A[(w - 1) * w + (w - 1)];
        s.e[w - 1] = 0.0;
        s.beta[w - 1] = 0.0;
    }
    if (blockIdx.x == 0)
        for (int64_t jj = (w >= 2 ? w - 2 : 0); jj < w; ++jj)
            for (int64_t i = tid; i < w; i += blockDim.x) s.Uh[jj * w + i] = 0.0;
}

// Two block sums with one pair of barriers (same per-value order as block_sum).
__device__ void block_sum2(double& a, double& b, double* red2) {
    a = warp_sum(a);
    b = warp_sum(b);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
    __syncthreads();
    if (lane == 0) {
        red2[warp] = a;
        red2[nw + warp] = b;
    }
    __syncthreads();
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < nw; ++i) {
        sa += red2[i];
        sb += red2[nw + i];
    }
    a = sa;
    b = sb;
}

// Householder vector of x[0..m) into u (skip: beta = 0, u = x); alpha out.
// Whole CTA, two block sums (the same arithmetic as k_tridiag's inline copy).
__device__ double tri_hh(const double* x, int64_t m, double* u, double* red, double& alpha, bool& skip) {
    const int tid = threadIdx.x;
    double ss = 0.0, tail = 0.0;
    for (int64_t i = tid; i < m; i += blockDim.x) {
        const double v = x[i];
        u[i] = v;
        ss += v * v;
        if (i > 0) tail += v * v;
    }
    block_sum2(ss, tail, red);  // red holds 2 x (warps) doubles
    const double x0 = u[0];
    skip = !(tail > 0.0);
    alpha = x0;
    double beta = 0.0;
    if (!skip) {
        const double nrm = sqrt(ss);
        alpha = x0 >= 0.0 ? -nrm : nrm;
        const double u0 = x0 - alpha;
        beta = 2.0 / (tail + u0 * u0);
        __syncthreads();
        if (tid == 0) u[0] = u0;
    }
    __syncthreads();
    return beta;
}

// One grid barrier per column (k_tridiag takes two). After the barrier of
// column j every CTA holds p_j = beta_j A22 u_j; each CTA then redundantly
// forms q_j, the updated row j + 1 (nobody stores it: it leaves the trailing
// matrix) and from it u_{j+1}; one fused pass per trailing row applies the
// rank-2 update of column j and dots the updated row with u_{j+1}, giving
// p_{j+1} for the next barrier (p double-buffered). Every entry sees the
// same operations in the same order as in k_tridiag, so d, e, beta and the
// reflectors are bitwise identical; the matrix is read and written once per
// column instead of read twice and written once.
__global__ void __launch_bounds__(kTriThreads, 1) k_tridiag1(TriState s) {
    extern __shared__ double sh[];
    const int64_t w = s.w;  // >= 4
    double* u = sh;           // u_j      (entries for columns j+1 ..)
    double* q = sh + w;       // q_j
    double* rn = sh + 2 * w;  // row j+1 of A^(j+1), columns j+1 ..
    double* un = sh + 3 * w;  // u_{j+1}  (entries for columns j+2 ..)
    __shared__ double red[2 * (kTriThreads / 32)];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + tid) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double* pc = s.p;   // p_j
    double* pn = s.p2;  // p_{j+1}
    double alpha;
    bool skip;
    double beta = tri_hh(s.A + 1, w - 1, u, red, alpha, skip);
    if (blockIdx.x == 0) {
        if (tid == 0) {
            s.d[0] = s.A[0];
            s.e[0] = alpha;
            s.beta[0] = beta;
        }
        for (int64_t i = tid; i < w; i += blockDim.x) s.Uh[i] = (i > 0 && !skip) ? u[i - 1] : 0.0;
    }
    // p_0 = beta_0 A22 u_0
    for (int64_t r = gwarp; r < w - 1; r += nwarps) {
        const double* ar = s.A + (1 + r) * w + 1;
        double acc = 0.0;
        for (int64_t c = lane; c < w - 1; c += 32) acc = fma(ar[c], u[c], acc);
        acc = warp_sum(acc);
        if (lane == 0) pc[r] = beta * acc;
    }
    grid_barrier(s.bar, gridDim.x);
    for (int64_t j = 0; j + 2 < w; ++j) {
        const int64_t m = w - j - 1;
        const bool last = j + 3 == w;
        // q_j = p_j - (beta_j / 2)(u_j . p_j) u_j
        double kk = 0.0;
        for (int64_t i = tid; i < m; i += blockDim.x) {
            const double pv = pc[i];
            q[i] = pv;
            kk += u[i] * pv;
        }
        kk = 0.5 * beta * block_sum(kk, red);
        for (int64_t i = tid; i < m; i += blockDim.x) q[i] -= kk * u[i];
        __syncthreads();
        // row j+1 after column j's update
        const double* rowo = s.A + (j + 1) * w + (j + 1);
        const double u0 = u[0], q0 = q[0];
        for (int64_t c = tid; c < m; c += blockDim.x) rn[c] = rowo[c] - (u0 * q[c] + q0 * u[c]);
        __syncthreads();
        double beta_n = 0.0;
        if (!last) {
            double alpha_n;
            bool skip_n;
            beta_n = tri_hh(rn + 1, m - 1, un, red, alpha_n, skip_n);
            if (blockIdx.x == 0) {
                if (tid == 0) {
                    s.d[j + 1] = rn[0];
                    s.e[j + 1] = alpha_n;
                    s.beta[j + 1] = beta_n;
                }
                double* uh = s.Uh + (j + 1) * w;
                for (int64_t i = tid; i < w; i += blockDim.x) uh[i] = (i > j + 1 && !skip_n) ? un[i - j - 2] : 0.0;
            }
        } else if (blockIdx.x == 0 && tid == 0) {
            s.d[j + 1] = rn[0];
            s.e[j + 1] = rn[1];
            s.beta[j + 1] = 0.0;
        }
        // rows j+2 .. : update (columns j+2 ..) fused with the dot against u_{j+1}
        for (int64_t rr = gwarp; rr < m - 1; rr += nwarps) {
            double* ar = s.A + (j + 2 + rr) * w + (j + 2);
            const double ur = u[rr + 1], qr = q[rr + 1];
            double acc = 0.0;
            const int64_t mm = m - 1;
            int64_t cc = lane;
            // 8 independent L2 loads in flight per lane (the pass is latency
            // bound); the dot accumulates in column order as before
            for (; cc + 32 * 7 < mm; cc += 32 * 8) {
                double v[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) v[t] = ar[cc + 32 * t];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int64_t c = cc + 32 * t;
                    v[t] = v[t] - (ur * q[c + 1] + qr * u[c + 1]);
                    ar[c] = v[t];
                    if (!last) acc = fma(v[t], un[c], acc);
                }
            }
            for (; cc < mm; cc += 32) {
                const double v = ar[cc] - (ur * q[cc + 1] + qr * u[cc + 1]);
                ar[cc] = v;
                if (!last) acc = fma(v, un[cc], acc);
            }
            if (!last) {
                acc = warp_sum(acc);
                if (lane == 0) pn[rr] = beta_n * acc;
            }
        }
        grid_barrier(s.bar, gridDim.x);
        double* t = u;
        u = un;
        un = t;
        t = pc;
        pc = pn;
        pn = t;
        beta = beta_n;
    }
    if (blockIdx.x == 0) {
        if (tid == 0) {
            s.d[w - 1] = s.A[(w - 1) * w + (w - 1)];
            s.e[w - 1] = 0.0;
            s.beta[w - 1] = 0.0;
        }
        for (int64_t jj = w - 2; jj < w; ++jj)
            for (int64_t i = tid; i < w; i += blockDim.x) s.Uh[jj * w + i] = 0.0;
    }
}

// k_tridiag1 with the matrix distributed over the CTAs' shared memory (row r
// in CTA r % G): the fused update+matvec pass reads shared memory instead of
// L2. The one row every CTA needs from another (row j+1 at column j) is
// published to global memory by its owner in the pass that last updates it;
// p goes through global memory as before. For w where the rows fit
// (ceil(w / G) * w doubles plus 4 w of vectors), else k_tridiag1.
__global__ void __launch_bounds__(kTriThreads, 1) k_tridiag_sm(TriState s) {
    extern __shared__ double sh[];
    const int64_t w = s.w;  // >= 4
    const int G = gridDim.x, rank = blockIdx.x;
    const int nloc = (int)((w + G - 1) / G);
    double* Aloc = sh;                         // nloc x w
    double* u = Aloc + (size_t)nloc * w;       // u_j
    double* q = u + w;                         // q_j
    double* rn = q + w;                        // row j+1 of A^(j+1)
    double* un = rn + w;                       // u_{j+1}
    __shared__ double red[2 * (kTriThreads / 32)];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kTriThreads / 32;
    for (int lr = 0; lr < nloc; ++lr) {
        const int64_t r = rank + (int64_t)G * lr;
        for (int64_t c = tid; c < w; c += kTriThreads) Aloc[(size_t)lr * w + c] = r < w ? s.A[r * w + c] : 0.0;
    }
    double* pc = s.p;
    double* pn = s.p2;
    double alpha;
    bool skip;
    double beta = tri_hh(s.A + 1, w - 1, u, red, alpha, skip);
    if (rank == 0) {
        if (tid == 0) {
            s.d[0] = s.A[0];
            s.e[0] = alpha;
            s.beta[0] = beta;
        }
        for (int64_t i = tid; i < w; i += kTriThreads) s.Uh[i] = (i > 0 && !skip) ? u[i - 1] : 0.0;
    }
    {
        const int lr0 = rank >= 1 ? 0 : 1;  // rows r >= 1
        for (int lr = lr0 + warp; lr < nloc; lr += nw) {
            const int64_t r = rank + (int64_t)G * lr;
            if (r >= w) break;
            const double* ar = Aloc + (size_t)lr * w + 1;
            double acc = 0.0;
            for (int64_t c = lane; c < w - 1; c += 32) acc = fma(ar[c], u[c], acc);
            acc = warp_sum(acc);
            if (lane == 0) pc[r - 1] = beta * acc;
        }
    }
    grid_barrier(s.bar, gridDim.x);
    for (int64_t j = 0; j + 2 < w; ++j) {
        const int64_t m = w - j - 1;
        const bool last = j + 3 == w;
        // p_j and row j+1 (published) from L2, loads issued together
        constexpr int kPer = 4;  // w <= kPer * kTriThreads
        double rowv[kPer];
        const double* rowo = s.A + (j + 1) * w + (j + 1);
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int64_t c = tid + (int64_t)t * kTriThreads;
            rowv[t] = c < m ? __ldcg(rowo + c) : 0.0;
        }
        double kk = 0.0;
        for (int64_t i = tid; i < m; i += kTriThreads) {
            const double pv = __ldcg(pc + i);
            q[i] = pv;
            kk += u[i] * pv;
        }
        kk = 0.5 * beta * block_sum(kk, red);
        for (int64_t i = tid; i < m; i += kTriThreads) q[i] -= kk * u[i];
        __syncthreads();
        {
            const double u0 = u[0], q0 = q[0];
#pragma unroll
            for (int t = 0; t < kPer; ++t) {
                const int64_t c = tid + (int64_t)t * kTriThreads;
                if (c < m) rn[c] = rowv[t] - (u0 * q[c] + q0 * u[c]);
            }
        }
        __syncthreads();
        double beta_n = 0.0;
        if (!last) {
            double alpha_n;
            bool skip_n;
            beta_n = tri_hh(rn + 1, m - 1, un, red, alpha_n, skip_n);
            if (rank == 0) {
                if (tid == 0) {
                    s.d[j + 1] = rn[0];
                    s.e[j + 1] = alpha_n;
                    s.beta[j + 1] = beta_n;
                }
                double* uh = s.Uh + (j + 1) * w;
                for (int64_t i = tid; i < w; i += kTriThreads) uh[i] = (i > j + 1 && !skip_n) ? un[i - j - 2] : 0.0;
            }
        } else if (rank == 0 && tid == 0) {
            s.d[j + 1] = rn[0];
            s.e[j + 1] = rn[1];
            s.beta[j + 1] = 0.0;
        }
        // own rows j+2 ..: update + dot with u_{j+1}; row j+2 is published
        const int64_t first = j + 2;
        const int lr0 = (int)((first - rank + G - 1) / G);
        for (int lr = (lr0 > 0 ? lr0 : 0) + warp; lr < nloc; lr += nw) {
            const int64_t r = rank + (int64_t)G * lr;
            if (r >= w) break;
            double* ar = Aloc + (size_t)lr * w + (j + 2);
            const int64_t ir = r - j - 1;
            const double ur = u[ir], qr = q[ir];
            const bool pub = r == j + 2;
            double* gout = s.A + r * w + (j + 2);
            double acc = 0.0;
            for (int64_t cc = lane; cc < m - 1; cc += 32) {
                const double v = ar[cc] - (ur * q[cc + 1] + qr * u[cc + 1]);
                ar[cc] = v;
                if (pub) gout[cc] = v;
                if (!last) acc = fma(v, un[cc], acc);
            }
            if (!last) {
                acc = warp_sum(acc);
                if (lane == 0) pn[r - j - 2] = beta_n * acc;
            }
        }
        grid_barrier(s.bar, gridDim.x);
        double* t = u;
        u = un;
        un = t;
        t = pc;
        pc = pn;
        pn = t;
        beta = beta_n;
    }
    if (rank == (int)((w - 1) % G) && tid == 0) {
        s.d[w - 1] = Aloc[(size_t)((w - 1) / G) * w + (w - 1)];
        s.e[w - 1] = 0.0;
        s.beta[w - 1] = 0.0;
    }
    if (rank == 0)
        for (int64_t jj = w - 2; jj < w; ++jj)
            for (int64_t i = tid; i < w; i += kTriThreads) s.Uh[jj * w + i] = 0.0;
}

// Cluster-resident tridiagonalisation (w <= kClTriMaxW): the whole w x w
// matrix lives in the distributed shared memory of one cluster of kClTri
// CTAs (row r in CTA r % kClTri), so a column step costs two cluster
// barriers instead of two grid barriers plus L2 round trips (w = 600: 4.1 ms
// vs 5.6 ms for k_tridiag). Per column j:
//   owner of row j: Householder vector of A[j, j+1:] (as k_tridiag);
//   barrier; every CTA copies u over DSMEM, computes p = beta A22 u for its
//   rows; barrier; every CTA gathers p over DSMEM, forms q = p - (beta/2)
//   (u.p) u and applies A22 -= u q^T + q u^T to its rows.
// u and p are double-buffered by column parity, so the next column's writes
// never race with this column's remote reads. (Measured alternatives, not
// faster: pushing u / p with remote stores, 4.2 ms; the matrix in registers
// across the cluster, 4.3 ms — the per-column cost is the local matrix sweep,
// shared-memory bandwidth bound, plus the owner's reduction.)
constexpr int kClTri = 16;
constexpr int kClTriThreads = 512;
constexpr int kClTriMaxW = 608;
constexpr int kClRegs = (kClTriMaxW + 31) / 32;  // u / q entries per lane

// Householder vector of row j (entries j+1 .. w-1 of the current row, `rowj`
// points at entry j+1; m = w - j - 1) into u, scalars (beta, alpha, skip) into
// sc, and the step's d / e / beta / Uh outputs. Whole CTA (two block sums).
__device__ void cl_householder(TriState& s, int j, int m, const double* rowj, double dj, double* u, double* sc,
                               double* red) {
    const int tid = threadIdx.x, w = (int)s.w;
    double ss = 0.0, tail = 0.0;
    for (int i = tid; i < m; i += kClTriThreads) {
        const double x = rowj[i];
        u[i] = x;
        ss += x * x;
        if (i > 0) tail += x * x;
    }
    ss = block_sum(ss, red);
    tail = block_sum(tail, red);
    const double x0 = u[0];
    const bool skip = !(tail > 0.0);
    double alpha = x0, beta = 0.0;
    if (!skip) {
        const double nrm = sqrt(ss);
        alpha = x0 >= 0.0 ? -nrm : nrm;
        const double u0 = x0 - alpha;
        beta = 2.0 / (tail + u0 * u0);
        __syncthreads();
        if (tid == 0) u[0] = u0;
    }
    if (tid == 0) {
        sc[0] = beta;
        sc[1] = alpha;
        sc[2] = skip ? 1.0 : 0.0;
        s.d[j] = dj;
        s.e[j] = alpha;
        s.beta[j] = beta;
    }
    __syncthreads();
    double* uh = s.Uh + (size_t)j * w;
    for (int i = tid; i < w; i += kClTriThreads) uh[i] = (i > j && !skip) ? u[i - j - 1] : 0.0;
}

// Look-ahead: the owner of row j+1 applies column j's rank-2 update to that
// row first and computes the next Householder vector while the other CTAs
// are still updating their rows, so step j+1 starts with u already in place
// (one Householder computation off the per-column critical path).
__global__ void __launch_bounds__(kClTriThreads, 1) k_tridiag_cluster(TriState s) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ double sh[];
    const int w = (int)s.w;
    const int rank = (int)cluster.block_rank();
    const int nloc = (w + kClTri - 1) / kClTri;  // local rows: global r = rank + kClTri * lr
    double* Aloc = sh;                            // nloc x w
    double* ubuf = Aloc + (size_t)nloc * w;      // [2][w]
    double* pbuf = ubuf + 2 * w;                 // [2][w]  (indexed by global row)
    double* q = pbuf + 2 * w;                    // w
    __shared__ double red[kClTriThreads / 32];
    __shared__ double scal[2][4];                // per parity: beta, alpha, skip
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kClTriThreads / 32;
    for (int lr = 0; lr < nloc; ++lr) {
        const int r = rank + kClTri * lr;
        for (int c = tid; c < w; c += kClTriThreads) Aloc[(size_t)lr * w + c] = r < w ? s.A[(size_t)r * w + c] : 0.0;
    }
    __syncthreads();
    if (w > 2 && rank == 0)  // step 0's vector (row 0 lives in CTA 0)
        cl_householder(s, 0, w - 1, Aloc + 1, Aloc[0], ubuf, &scal[0][0], red);
    for (int j = 0; j + 2 < w; ++j) {
        const int par = j & 1;
        const int m = w - j - 1;
        double* u = ubuf + par * w;      // u[0..m): entries for columns j+1 ..
        double* pp = pbuf + par * w;
        const int owner = j % kClTri;
        const int nxt = (j + 1) % kClTri;                 // owner of row j+1
        const bool look = j + 3 < w && rank == nxt;       // computes step j+1's vector here
        double* un = ubuf + (par ^ 1) * w;
        double* rown = Aloc + (size_t)((j + 1) / kClTri) * w + (j + 1);  // row j+1 from column j+1 (nxt only)
        cluster.sync();
        // fetch u and the scalars from the owner (DSMEM)
        const double* uo = cluster.map_shared_rank(u, owner);
        const double* so = cluster.map_shared_rank(&scal[par][0], owner);
        const double beta = so[0];
        const bool skip = so[2] != 0.0;
        if (skip) {  // uniform: row j is already reduced; row j+1 is unchanged
            if (look) cl_householder(s, j + 1, m - 1, rown + 1, rown[0], un, &scal[par ^ 1][0], red);
            continue;
        }
        if (rank != owner)
            for (int i = tid; i < m; i += kClTriThreads) u[i] = uo[i];
        __syncthreads();
        // p_r = beta * A22[r, :] . u for this CTA's trailing rows (warp per row);
        // lane l touches columns l + 32 i of every row, so its u entries stay in
        // registers (one shared-memory read per matrix element instead of two)
        const int lr0 = (j + 1 - rank + kClTri - 1) / kClTri;  // first local row with global r > j
        double ureg[kClRegs];
#pragma unroll
        for (int i = 0; i < kClRegs; ++i) ureg[i] = lane + 32 * i < m ? u[lane + 32 * i] : 0.0;
        for (int lr = lr0 + warp; lr < nloc; lr += nw) {
            const int r = rank + kClTri * lr;
            if (r >= w) break;
            const double* ar = Aloc + (size_t)lr * w + (j + 1);
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < kClRegs; ++i)
                if (lane + 32 * i < m) acc = fma(ar[lane + 32 * i], ureg[i], acc);
            acc = warp_sum(acc);
            if (lane == 0) pp[r] = beta * acc;
        }
        cluster.sync();
        // gather p (row i lives in CTA i % kClTri), kk = beta/2 u.p, q = p - kk u
        double kk = 0.0;
        for (int i = tid; i < m; i += kClTriThreads) {
            const int r = j + 1 + i;
            const double* pr = cluster.map_shared_rank(pp, r % kClTri);
            const double pv = pr[r];
            q[i] = pv;
            kk += u[i] * pv;
        }
        kk = 0.5 * beta * block_sum(kk, red);
        for (int i = tid; i < m; i += kClTriThreads) q[i] -= kk * u[i];
        __syncthreads();
        if (look) {  // row j+1 first (ir = 0), then its Householder vector
            const double u0 = u[0], q0 = q[0];
            for (int c = tid; c < m; c += kClTriThreads) rown[c] -= u0 * q[c] + q0 * u[c];
            __syncthreads();
            cl_householder(s, j + 1, m - 1, rown + 1, rown[0], un, &scal[par ^ 1][0], red);
        }
        double qreg[kClRegs];
#pragma unroll
        for (int i = 0; i < kClRegs; ++i) qreg[i] = lane + 32 * i < m ? q[lane + 32 * i] : 0.0;
        for (int lr = lr0 + warp; lr < nloc; lr += nw) {
            const int r = rank + kClTri * lr;
            if (r >= w) break;
            if (look && r == j + 1) continue;  // done above
            double* ar = Aloc + (size_t)lr * w + (j + 1);
            const int ir = r - j - 1;
            const double ur = u[ir], qr = q[ir];
#pragma unroll
            for (int i = 0; i < kClRegs; ++i)
                if (lane + 32 * i < m) ar[lane + 32 * i] -= ur * qreg[i] + qr * ureg[i];
        }
        __syncthreads();
    }
    // last 2 x 2 block
    const int jl = w >= 2 ? w - 2 : 0;
    for (int jj = jl; jj < w; ++jj) {
        if (rank == jj % kClTri && tid == 0) {
            const double* rr = Aloc + (size_t)(jj / kClTri) * w;
            s.d[jj] = rr[jj];
            s.e[jj] = jj + 1 < w ? rr[jj + 1] : 0.0;
            s.beta[jj] = 0.0;
        }
    }
    if (rank == 0)
        for (int jj = jl; jj < w; ++jj)
            for (int i = tid; i < w; i += kClTriThreads) s.Uh[(size_t)jj * w + i] = 0.0;
    cluster.sync();  // keep every CTA's shared memory alive until remote reads are done
}

// One cluster barrier per column (k_tridiag_cluster takes two), the
// k_tridiag1 scheme on distributed shared memory: after the barrier of
// column j every CTA gathers p_j, forms q_j, reads row j + 1 from its owner
// (nobody updates that row in column j: it leaves the trailing matrix) and
// builds u_{j+1} itself; then one pass over its trailing rows applies the
// rank-2 update and dots each updated row with u_{j+1}, leaving p_{j+1} for
// the next barrier. u, p double-buffered by column parity.
__global__ void __launch_bounds__(kClTriThreads, 1) k_tridiag_cluster1(TriState s) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ double sh[];
    const int w = (int)s.w;  // >= 4
    const int rank = (int)cluster.block_rank();
    const int nloc = (w + kClTri - 1) / kClTri;
    double* Aloc = sh;                        // nloc x w
    double* ubuf = Aloc + (size_t)nloc * w;  // [2][w]
    double* pbuf = ubuf + 2 * w;             // [2][w]  (indexed by global row)
    double* q = pbuf + 2 * w;                // w
    double* rn = q + w;                      // w
    __shared__ double red[2 * (kClTriThreads / 32)];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kClTriThreads / 32;
    for (int lr = 0; lr < nloc; ++lr) {
        const int r = rank + kClTri * lr;
        for (int c = tid; c < w; c += kClTriThreads) Aloc[(size_t)lr * w + c] = r < w ? s.A[(size_t)r * w + c] : 0.0;
    }
    cluster.sync();
    // column 0: every CTA forms u_0 from row 0 (CTA 0) and p_0 for its rows
    double beta;
    {
        const double* row0 = cluster.map_shared_rank(Aloc, 0);
        for (int c = tid; c < w; c += kClTriThreads) rn[c] = row0[c];
        __syncthreads();
        double alpha;
        bool skip;
        beta = tri_hh(rn + 1, w - 1, ubuf, red, alpha, skip);
        if (rank == 0) {
            if (tid == 0) {
                s.d[0] = rn[0];
                s.e[0] = alpha;
                s.beta[0] = beta;
            }
            for (int i = tid; i < w; i += kClTriThreads) s.Uh[i] = (i > 0 && !skip) ? ubuf[i - 1] : 0.0;
        }
        const int lr0 = (1 - rank + kClTri - 1) / kClTri;
        for (int lr = lr0 + warp; lr < nloc; lr += nw) {
            const int r = rank + kClTri * lr;
            if (r >= w) break;
            const double* ar = Aloc + (size_t)lr * w + 1;
            double acc = 0.0;
            for (int c = lane; c < w - 1; c += 32) acc = fma(ar[c], ubuf[c], acc);
            acc = warp_sum(acc);
            if (lane == 0) pbuf[r] = beta * acc;
        }
    }
    cluster.sync();
    for (int j = 0; j + 2 < w; ++j) {
        const int par = j & 1;
        const int m = w - j - 1;
        const bool last = j + 3 == w;
        double* u = ubuf + par * w;
        double* un = ubuf + (par ^ 1) * w;
        double* pp = pbuf + par * w;
        double* pn = pbuf + (par ^ 1) * w;
        // q_j from the gathered p_j; row j+1 (owner's smem) fetched alongside
        constexpr int kRowPer = (kClTriMaxW + kClTriThreads - 1) / kClTriThreads;
        double rowv[kRowPer];
        {
            const double* ro = cluster.map_shared_rank(Aloc + (size_t)((j + 1) / kClTri) * w + (j + 1), (j + 1) % kClTri);
#pragma unroll
            for (int t = 0; t < kRowPer; ++t) {
                const int c = tid + t * kClTriThreads;
                rowv[t] = c < m ? ro[c] : 0.0;
            }
        }
        double kk = 0.0;
        for (int i = tid; i < m; i += kClTriThreads) {
            const int r = j + 1 + i;
            const double* pr = cluster.map_shared_rank(pp, r % kClTri);
            const double pv = pr[r];
            q[i] = pv;
            kk += u[i] * pv;
        }
        kk = 0.5 * beta * block_sum(kk, red);
        for (int i = tid; i < m; i += kClTriThreads) q[i] -= kk * u[i];
        __syncthreads();
        // row j+1 after column j's update
        {
            const double u0 = u[0], q0 = q[0];
#pragma unroll
            for (int t = 0; t < kRowPer; ++t) {
                const int c = tid + t * kClTriThreads;
                if (c < m) rn[c] = rowv[t] - (u0 * q[c] + q0 * u[c]);
            }
        }
        __syncthreads();
        double beta_n = 0.0;
        if (!last) {
            double alpha_n;
            bool skip_n;
            beta_n = tri_hh(rn + 1, m - 1, un, red, alpha_n, skip_n);
            if (rank == 0) {
                if (tid == 0) {
                    s.d[j + 1] = rn[0];
                    s.e[j + 1] = alpha_n;
                    s.beta[j + 1] = beta_n;
                }
                double* uh = s.Uh + (size_t)(j + 1) * w;
                for (int i = tid; i < w; i += kClTriThreads) uh[i] = (i > j + 1 && !skip_n) ? un[i - j - 2] : 0.0;
            }
        } else if (rank == 0 && tid == 0) {
            s.d[j + 1] = rn[0];
            s.e[j + 1] = rn[1];
            s.beta[j + 1] = 0.0;
        }
        // fused pass over this CTA's rows j+2 ..; lane l handles columns
        // j+2+l+32i, so its q / u_{j+1} entries sit in registers (u from smem)
        double qreg[kClRegs], nreg[kClRegs];
#pragma unroll
        for (int i = 0; i < kClRegs; ++i) {
            const int c = lane + 32 * i;
            qreg[i] = c < m - 1 ? q[c + 1] : 0.0;
            nreg[i] = (c < m - 1 && !last) ? un[c] : 0.0;
        }
        const int lr0 = (j + 2 - rank + kClTri - 1) / kClTri;  // first local row with global r > j + 1
        for (int lr = lr0 + warp; lr < nloc; lr += nw) {
            const int r = rank + kClTri * lr;
            if (r >= w) break;
            double* ar = Aloc + (size_t)lr * w + (j + 2);
            const int ir = r - j - 1;
            const double ur = u[ir], qr = q[ir];
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < kClRegs; ++i) {
                const int c = lane + 32 * i;
                if (c < m - 1) {
                    const double v = ar[c] - (ur * qreg[i] + qr * u[c + 1]);
                    ar[c] = v;
                    acc = fma(v, nreg[i], acc);
                }
            }
            if (!last) {
                acc = warp_sum(acc);
                if (lane == 0) pn[r] = beta_n * acc;
            }
        }
        beta = beta_n;
        cluster.sync();
    }
    if (rank == (w - 1) % kClTri && tid == 0) {
        s.d[w - 1] = Aloc[(size_t)((w - 1) / kClTri) * w + (w - 1)];
        s.e[w - 1] = 0.0;
        s.beta[w - 1] = 0.0;
    }
    if (rank == 0)
        for (int jj = w - 2; jj < w; ++jj)
            for (int i = tid; i < w; i += kClTriThreads) s.Uh[(size_t)jj * w + i] = 0.0;
    cluster.sync();  // keep every CTA's shared memory alive until remote reads are done
}

__global__ void k_copy_sym(int64_t w, const double* __restrict__ M, int64_t ldm, double* __restrict__ A) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= w * w) return;
    int64_t i = e / w, j = e % w;
    A[e] = 0.5 * (M[i * ldm + j] + M[j * ldm + i]);
}

// Gershgorin bounds, ||T||_1 and pivmin (dstebz), one CTA.
__global__ void k_tri_bounds(int64_t w, const double* __restrict__ d, const double* __restrict__ e,
                             double* __restrict__ out) {
    __shared__ double rlo[32], rhi[32], rn[32], re2[32];
    double lo = 1e300, hi = -1e300, nrm = 0.0, emax2 = 0.0;
    for (int64_t i = threadIdx.x; i < w; i += blockDim.x) {
        const double em = i > 0 ? fabs(e[i - 1]) : 0.0;
        const double ep = i + 1 < w ? fabs(e[i]) : 0.0;
        lo = fmin(lo, d[i] - em - ep);
        hi = fmax(hi, d[i] + em + ep);
        nrm = fmax(nrm, fabs(d[i]) + em + ep);
        if (i + 1 < w) emax2 = fmax(emax2, e[i] * e[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
        emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
    }
    const int wp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        rlo[wp] = lo;
        rhi[wp] = hi;
        rn[wp] = nrm;
        re2[wp] = emax2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            lo = fmin(lo, rlo[i]);
            hi = fmax(hi, rhi[i]);
            nrm = fmax(nrm, rn[i]);
            emax2 = fmax(emax2, re2[i]);
        }
        lo = fmin(lo, rlo[0]);
        hi = fmax(hi, rhi[0]);
        nrm = fmax(nrm, rn[0]);
        emax2 = fmax(emax2, re2[0]);
        const double tnorm = fmax(fabs(lo), fabs(hi));
        const double eps = 2.220446049250313e-16;
        out[0] = lo - 2.0 * eps * tnorm - 1e-300;
        out[1] = hi + 2.0 * eps * tnorm + 1e-300;
        out[2] = nrm;
        out[3] = 2.2250738585072014e-308 * fmax(1.0, emax2);  // pivmin
    }
}

// number of eigenvalues of T strictly below x (Sturm count with pivmin guard)
__global__ void k_e2(int64_t w, const double* __restrict__ e, double* __restrict__ e2) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < w) e2[i] = e[i] * e[i];
}

// 1/q for the Sturm recurrence: the approximate FP64 reciprocal refined by two
// Newton steps (a few ulp; the count is then exact for a tridiagonal within a
// few ulp of T, the same backward-error class as with IEEE division, which
// costs ~3x the instructions on this issue-bound recurrence).
__device__ __forceinline__ double sturm_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    return fma(r, e, r);
}

// NS Sturm sequences evaluated together (independent division chains: the
// recurrence is latency bound, so interleaving hides most of it).
#ifndef RSVD_STURM_DIV
#define RSVD_STURM_DIV 0
#endif
template <int NS>
__device__ __forceinline__ void sturm_count_n(int64_t w, const double* __restrict__ d, const double* __restrict__ e2,
                                              const double* x, double pivmin, int* cnt) {
    double qv[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
        qv[t] = d[0] - x[t];
        if (fabs(qv[t]) < pivmin) qv[t] = -pivmin;
        cnt[t] = qv[t] < 0.0;
    }
    for (int64_t i = 1; i < w; ++i) {
        const double di = d[i], ei = e2[i - 1];
#pragma unroll
        for (int t = 0; t < NS; ++t) {
            qv[t] = (di - x[t]) - ei * (RSVD_STURM_DIV ? 1.0 / qv[t] : sturm_rcp(qv[t]));
            if (fabs(qv[t]) < pivmin) qv[t] = -pivmin;
            cnt[t] += qv[t] < 0.0;
        }
    }
}

// eigenvalue number `idx` in ascending order; one warp per eigenvalue,
// 32 x kMsShifts Sturm counts per step (multisection: the bracket shrinks by
// 32 kMsShifts + 1 per step).
constexpr int kMsShifts = 1;  // 2 and 4 measured slower (w = 600: 4.6 -> 5.6 ms at 4): the divisions are issue bound

__global__ void k_multisect(int64_t w, int64_t k, const double* __restrict__ d, const double* __restrict__ e2,
                            const double* __restrict__ bounds, double* __restrict__ evals) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= k) return;
    constexpr int NP = 32 * kMsShifts;  // points per step
    const int64_t target = w - 1 - wid;  // wid-th largest
    double lo = bounds[0], hi = bounds[1];
    const double pivmin = bounds[3];
    const double eps = 2.220446049250313e-16;
    for (int it = 0; it < 64; ++it) {
        const double width = hi - lo;
        if (!(width > 2.0 * eps * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin)) break;
        double x[kMsShifts];
        int c[kMsShifts];
#pragma unroll
        for (int t = 0; t < kMsShifts; ++t) x[t] = lo + width * (double)(lane + 32 * t + 1) / (double)(NP + 1);
        sturm_count_n<kMsShifts>(w, d, e2, x, pivmin, c);
        // count(x) <= target  <=>  eigenvalue #target is >= x; counts are
        // monotone in x, so points 0 .. nb-1 satisfy
        int nb = 0;
#pragma unroll
        for (int t = 0; t < kMsShifts; ++t) nb += __popc(__ballot_sync(0xffffffffu, c[t] <= target));
        const double nlo = nb > 0 ? lo + width * (double)nb / (double)(NP + 1) : lo;
        const double nhi = nb < NP ? lo + width * (double)(nb + 1) / (double)(NP + 1) : hi;
        lo = nlo;
        hi = nhi;
    }
    if (lane == 0) evals[wid] = 0.5 * (lo + hi);
}

__global__ void k_clusters(int64_t k, const double* __restrict__ evals, const double* __restrict__ bounds,
                           int32_t* __restrict__ cstart, int32_t* __restrict__ ncl) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    // eigenvectors of eigenvalues separated by more than ortol come out of
    // inverse iteration orthogonal to ~2 eps ||T|| / gap <= 5e-11 already; only
    // closer ones are chained through MGS (dstein uses 1e-3 ||T||).
    const double ortol = bounds[2] > 0.0 ? 1e-5 * bounds[2] : 1e300;  // T = 0: one cluster
    int n = 0;
    for (int64_t i = 0; i < k; ++i)
        if (i == 0 || evals[i - 1] - evals[i] > ortol) cstart[n++] = (int32_t)i;
    cstart[n] = (int32_t)k;
    ncl[0] = n;
}

__device__ __forceinline__ double init_vec(int64_t i, int64_t member) {
    uint64_t z = (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ULL ^ (uint64_t)(member + 7) * 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

// One warp per cluster. For each member: pivoted LU of T - lambda I (lane 0,
// reciprocal pivots), 3 inverse-iteration solves, each followed by MGS against
// the cluster's earlier vectors and normalisation (whole warp).
__global__ void k_invit(int64_t w, int64_t k, const double* __restrict__ d, const double* __restrict__ e,
                        const double* __restrict__ evals, const double* __restrict__ bounds,
                        const int32_t* __restrict__ cstart, const int32_t* __restrict__ ncl,
                        double* __restrict__ X /* k x w, row = vector */, double* __restrict__ fac /* per warp 5w */,
                        int32_t* __restrict__ info) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= ncl[0]) return;
    const int64_t c0 = cstart[wid], c1 = cstart[wid + 1];
    double* u0 = fac + wid * 5 * w;  // reciprocal of U diagonal
    double* u1 = u0 + w;
    double* u2 = u1 + w;
    double* l = u2 + w;
    double* sw = l + w;  // swap flags (0/1 as double)
    const double tnorm = bounds[2];
    // ||T|| = 0 (zero Rayleigh-Ritz matrix, e.g. A = 0): every vector is an
    // eigenvector; unit pivots keep the iteration finite
    const double tiny = tnorm > 0.0 ? 2.220446049250313e-16 * tnorm : 1.0;
    for (int64_t mbr = c0; mbr < c1; ++mbr) {
        double* x = X + mbr * w;
        // perturb repeated eigenvalues slightly so the shifts differ (dstein)
        const double lam = evals[mbr] + (double)(mbr - c0) * 10.0 * tiny;
        if (lane == 0) {
            double cp = d[0] - lam, cq = w > 1 ? e[0] : 0.0, cr = 0.0;
            for (int64_t i = 0; i + 1 < w; ++i) {
                const double ci = e[i];
                const double an = d[i + 1] - lam, bn = (i + 2 < w) ? e[i + 1] : 0.0;
                if (fabs(ci) > fabs(cp)) {
                    const double r = 1.0 / ci;
                    const double mult = cp * r;
                    u0[i] = r;
                    u1[i] = an;
                    u2[i] = bn;
                    l[i] = mult;
                    sw[i] = 1.0;
                    cp = cq - mult * an;
                    cq = cr - mult * bn;
                } else {
                    const double piv = fabs(cp) < tiny ? (cp < 0.0 ? -tiny : tiny) : cp;
                    const double r = 1.0 / piv;
                    const double mult = ci * r;
                    u0[i] = r;
                    u1[i] = cq;
                    u2[i] = cr;
                    l[i] = mult;
                    sw[i] = 0.0;
                    cp = an - mult * cq;
                    cq = bn - mult * cr;
                }
                cr = 0.0;
            }
            const double piv = fabs(cp) < tiny ? (cp < 0.0 ? -tiny : tiny) : cp;
            u0[w - 1] = 1.0 / piv;
        }
        for (int64_t i = lane; i < w; i += 32) x[i] = init_vec(i, mbr);
        __syncwarp();
        for (int it = 0; it < 3; ++it) {
            if (lane == 0) {
                // y = L^{-1} P x (carry in a register; x[i+1] loads are independent)
                double carry = x[0];
                for (int64_t i = 0; i + 1 < w; ++i) {
                    double a = carry, b = x[i + 1];
                    if (sw[i] != 0.0) {
                        const double t = a;
                        a = b;
                        b = t;
                    }
                    x[i] = a;
                    carry = b - l[i] * a;
                }
                // U x = y (two carries)
                double c1 = carry * u0[w - 1], c2 = 0.0;
                x[w - 1] = c1;
                for (int64_t i = w - 2; i >= 0; --i) {
                    const double v = (x[i] - u1[i] * c1 - u2[i] * c2) * u0[i];
                    x[i] = v;
                    c2 = c1;
                    c1 = v;
                }
            }
            __syncwarp();
            // MGS against the earlier members of this cluster
            for (int64_t o = c0; o < mbr; ++o) {
                const double* y = X + o * w;
                double dot = 0.0;
                for (int64_t i = lane; i < w; i += 32) dot += y[i] * x[i];
                dot = warp_sum(dot);
                for (int64_t i = lane; i < w; i += 32) x[i] -= dot * y[i];
                __syncwarp();
            }
            double nn = 0.0;
            for (int64_t i = lane; i < w; i += 32) nn += x[i] * x[i];
            nn = warp_sum(nn);
            if (!(nn > 0.0) || !isfinite(nn)) {
                if (lane == 0) info[0] = 0;
                nn = 1.0;
            }
            const double inv = 1.0 / sqrt(nn);
            for (int64_t i = lane; i < w; i += 32) x[i] *= inv;
            __syncwarp();
        }
    }
}

// x <- H_0 H_1 ... H_{w-3} x for every vector, then write evecs[:, i]
// (w x k row-major, ld lde). A CTA serves kBtVec vectors (one warp each,
// the vector in registers: lane l holds entries l + 32 c); the Householder
// rows stream through shared memory in blocks of kBtRows rows, double
// buffered with cp.async, so the L2 latency is paid once per block and each
// row is read once per CTA instead of once per vector.
constexpr int kBtChunks = 64;  // w <= 2048
constexpr int kBtRows = 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}

// NC = register chunks per lane (w <= 32 NC, instantiated per width class so
// the unrolled loops carry no dead predicated chunks), VPB = vectors (warps)
// per CTA (small k: fewer vectors per CTA, more CTAs).
template <int NC, int VPB>
__global__ void __launch_bounds__(32 * VPB)
k_backtransform(int64_t w, int64_t k, const double* __restrict__ Uh, const double* __restrict__ beta,
                const double* __restrict__ X, double* __restrict__ evecs, int64_t lde) {
    constexpr int kBtChunks = NC;
    extern __shared__ __align__(16) double ubuf[];  // [2][kBtRows][wp]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t v = (int64_t)blockIdx.x * VPB + warp;
    const int nc = (int)((w + 31) / 32);
    const int64_t wp = (w + 1) & ~int64_t(1);  // rows padded to 16 bytes
    double x[kBtChunks];
#pragma unroll
    for (int c = 0; c < kBtChunks; ++c) {
        const int64_t i = lane + 32 * c;
        x[c] = (c < nc && v < k && i < w) ? X[v * w + i] : 0.0;
    }
    const int64_t jtop = w - 3;  // reflectors jtop .. 0, applied in that order
    if (jtop < 0) goto store;
    {
        const int64_t nblk = (jtop + kBtRows) / kBtRows;  // block b: rows jtop - b R - (R-1) .. jtop - b R
        // 16-byte copies of block b's rows into buffer b & 1 (rows whose index < 0 skipped)
        auto issue = [&](int64_t b) {
            double* dst = ubuf + (b & 1) * kBtRows * wp;
            const bool vec = (w % 2) == 0;
            for (int rr = 0; rr < kBtRows; ++rr) {
                const int64_t j = jtop - b * kBtRows - rr;
                if (j < 0) break;
                if (vec) {
                    for (int64_t i = 2 * threadIdx.x; i < w; i += 2 * blockDim.x)
                        cp_async16(dst + rr * wp + i, Uh + j * w + i);
                } else {
                    for (int64_t i = threadIdx.x; i < w; i += blockDim.x) dst[rr * wp + i] = Uh[j * w + i];
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        issue(0);
        for (int64_t b = 0; b < nblk; ++b) {
            if (b + 1 < nblk) {
                issue(b + 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();
            const double* blk = ubuf + (b & 1) * kBtRows * wp;
            for (int rr = 0; rr < kBtRows; ++rr) {
                const int64_t j = jtop - b * kBtRows - rr;
                if (j < 0) break;
                const double bj = beta[j];
                if (bj == 0.0) continue;
                const double* u = blk + rr * wp;
                double dot = 0.0;
#pragma unroll
                for (int c = 0; c < kBtChunks; ++c)
                    if (c < nc) {
                        const int64_t i = lane + 32 * c;
                        dot = fma(i < w ? u[i] : 0.0, x[c], dot);
                    }
                dot = warp_sum(dot) * bj;
#pragma unroll
                for (int c = 0; c < kBtChunks; ++c)
                    if (c < nc) {
                        const int64_t i = lane + 32 * c;
                        if (i < w) x[c] = fma(-dot, u[i], x[c]);
                    }
            }
            __syncthreads();  // buffer (b & 1) is refilled by issue(b + 2)
        }
    }
store:
    if (v < k) {
#pragma unroll
        for (int c = 0; c < kBtChunks; ++c) {
            const int64_t i = lane + 32 * c;
            if (c < nc && i < w) evecs[i * lde + v] = x[c];
        }
    }
}

// Blocked variant: the kBtRows reflectors of a staged block are applied to
// a vector together. With D_r = u_r . x (x at the block start, all r at
// once: kBtRows independent dot chains instead of one), the sequential
// product H_{r0} H_{r1} ... applied to x is x - sum_r c_r u_r with
//   c_r = beta_r (D_r - sum_{s<r} G_rs c_s),   G_rs = u_r . u_s,
// G precomputed per block by k_bt_gram. Same Householder product, more
// instruction-level parallelism per warp (the one-by-one form is a chain of
// dependent dot -> warp_sum -> axpy steps per reflector).
constexpr int kBtG = kBtRows * kBtRows;

__global__ void k_bt_gram(int64_t w, const double* __restrict__ Uh, double* __restrict__ G) {
    const int64_t jtop = w - 3;
    const int64_t b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* g = G + b * kBtG;
    for (int pr = warp; pr < kBtG; pr += nw) {
        const int r = pr / kBtRows, c = pr % kBtRows;
        const int64_t jr = jtop - b * kBtRows - r, jc = jtop - b * kBtRows - c;
        double acc = 0.0;
        if (c < r && jc >= 0 && jr >= 0) {
            const double* ur = Uh + jr * w;
            const double* uc = Uh + jc * w;
            for (int64_t i = lane; i < w; i += 32) acc = fma(ur[i], uc[i], acc);
            acc = warp_sum(acc);
        }
        if (lane == 0) g[pr] = acc;
    }
}

template <int NC, int VPB>
__global__ void __launch_bounds__(32 * VPB)
k_backtransform_blk(int64_t w, int64_t k, const double* __restrict__ Uh, const double* __restrict__ beta,
                    const double* __restrict__ G, const double* __restrict__ X, double* __restrict__ evecs,
                    int64_t lde) {
    extern __shared__ __align__(16) double ubuf[];  // [2][kBtRows][wp]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t v = (int64_t)blockIdx.x * VPB + warp;
    const int nc = (int)((w + 31) / 32);
    const int64_t wp = (w + 1) & ~int64_t(1);
    double x[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int64_t i = lane + 32 * c;
        x[c] = (c < nc && v < k && i < w) ? X[v * w + i] : 0.0;
    }
    const int64_t jtop = w - 3;
    if (jtop >= 0) {
        const int64_t nblk = (jtop + kBtRows) / kBtRows;
        auto issue = [&](int64_t b) {
            double* dst = ubuf + (b & 1) * kBtRows * wp;
            const bool vec = (w % 2) == 0;
            for (int rr = 0; rr < kBtRows; ++rr) {
                const int64_t j = jtop - b * kBtRows - rr;
                if (j < 0) break;
                if (vec) {
                    for (int64_t i = 2 * threadIdx.x; i < w; i += 2 * blockDim.x)
                        cp_async16(dst + rr * wp + i, Uh + j * w + i);
                } else {
                    for (int64_t i = threadIdx.x; i < w; i += blockDim.x) dst[rr * wp + i] = Uh[j * w + i];
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        issue(0);
        for (int64_t b = 0; b < nblk; ++b) {
            if (b + 1 < nblk) {
                issue(b + 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();
            const double* blk = ubuf + (b & 1) * kBtRows * wp;
            const int nr = (int)min((int64_t)kBtRows, jtop - b * kBtRows + 1);  // valid rows (uniform)
            double dd[kBtRows];
#pragma unroll
            for (int r = 0; r < kBtRows; ++r) dd[r] = 0.0;
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if (c < nc) {
                    const int64_t i = lane + 32 * c;
                    if (i < w) {
#pragma unroll
                        for (int r = 0; r < kBtRows; ++r)
                            if (r < nr) dd[r] = fma(blk[r * wp + i], x[c], dd[r]);
                    }
                }
#pragma unroll
            for (int r = 0; r < kBtRows; ++r) dd[r] = warp_sum(dd[r]);
            const double* g = G + b * kBtG;
            double cf[kBtRows];
#pragma unroll
            for (int r = 0; r < kBtRows; ++r) {
                double t = dd[r];
#pragma unroll
                for (int s2 = 0; s2 < r; ++s2) t = fma(-g[r * kBtRows + s2], cf[s2], t);
                const int64_t j = jtop - b * kBtRows - r;
                cf[r] = r < nr ? beta[j] * t : 0.0;
            }
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if (c < nc) {
                    const int64_t i = lane + 32 * c;
                    if (i < w) {
                        double xc = x[c];
#pragma unroll
                        for (int r = 0; r < kBtRows; ++r)
                            if (r < nr) xc = fma(-cf[r], blk[r * wp + i], xc);
                        x[c] = xc;
                    }
                }
            __syncthreads();  // buffer (b & 1) is refilled by issue(b + 2)
        }
    }
    if (v < k) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int64_t i = lane + 32 * c;
            if (c < nc && i < w) evecs[i * lde + v] = x[c];
        }
    }
}

// Row-split blocked back-transformation: a CTA of 8 warps serves VPB vectors;
// warp ww owns rows [ww S, (ww + 1) S) of all of them (S = NCW x 32), so the
// FP64 pipe sees 8 warps per SM instead of one. Per block of kBtRows
// reflectors each lane loads its slice of the reflectors straight from L2
// (prefetched one block ahead, no shared-memory staging), forms partial dots
// for every (reflector, vector) pair, the CTA sums them (one round through
// shared memory), and every thread runs the kBtRows-step recurrence of
// k_backtransform_blk and applies the rank-kBtRows update to its rows.
constexpr int kRsWarps = 8;

template <int NCW, int VPB>
__global__ void __launch_bounds__(32 * kRsWarps)
k_backtransform_rs(int64_t w, int64_t k, const double* __restrict__ Uh, const double* __restrict__ beta,
                   const double* __restrict__ G, const double* __restrict__ X, double* __restrict__ evecs,
                   int64_t lde) {
    constexpr int R = kBtRows, NP = R * VPB;  // (reflector, vector) pairs
    __shared__ double red[kRsWarps][NP];
    __shared__ double dsum[NP];
    const int lane = threadIdx.x & 31, ww = threadIdx.x >> 5;
    const int64_t v0 = (int64_t)blockIdx.x * VPB;
    const int64_t S = (int64_t)NCW * 32;
    const int64_t i0 = ww * S + lane;
    double x[VPB][NCW];
#pragma unroll
    for (int v = 0; v < VPB; ++v)
#pragma unroll
        for (int c = 0; c < NCW; ++c) {
            const int64_t i = i0 + 32 * c;
            x[v][c] = (v0 + v < k && i < w) ? X[(v0 + v) * w + i] : 0.0;
        }
    const int64_t jtop = w - 3;
    const int64_t nblk = jtop >= 0 ? (jtop + R) / R : 0;
    // prefetch one block ahead when the registers allow it (NCW <= 4)
    constexpr bool PF = NCW <= 4;
    double u[R][NCW], un[PF ? R : 1][PF ? NCW : 1];
    auto load = [&](int64_t b, auto& dst) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t j = jtop - b * R - r;
#pragma unroll
            for (int c = 0; c < NCW; ++c) {
                const int64_t i = i0 + 32 * c;
                dst[r][c] = (j >= 0 && i < w) ? __ldg(Uh + j * w + i) : 0.0;
            }
        }
    };
    if (nblk > 0) load(0, u);
    for (int64_t b = 0; b < nblk; ++b) {
        if (PF) {
            if (b + 1 < nblk) load(b + 1, un);
        } else if (b > 0) {
            load(b, u);
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int v = 0; v < VPB; ++v) {
                double a = 0.0;
#pragma unroll
                for (int c = 0; c < NCW; ++c) a = fma(u[r][c], x[v][c], a);
                a = warp_sum(a);
                if (lane == 0) red[ww][r * VPB + v] = a;
            }
        __syncthreads();
        if (threadIdx.x < NP) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < kRsWarps; ++q) t += red[q][threadIdx.x];
            dsum[threadIdx.x] = t;
        }
        __syncthreads();
        const double* g = G + b * kBtG;
        const int nr = (int)min((int64_t)R, jtop - b * R + 1);
#pragma unroll
        for (int v = 0; v < VPB; ++v) {
            double cf[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double t = dsum[r * VPB + v];
#pragma unroll
                for (int s2 = 0; s2 < r; ++s2) t = fma(-g[r * R + s2], cf[s2], t);
                cf[r] = r < nr ? beta[jtop - b * R + (int64_t)(-r)] * t : 0.0;
            }
#pragma unroll
            for (int c = 0; c < NCW; ++c) {
                double xc = x[v][c];
#pragma unroll
                for (int r = 0; r < R; ++r) xc = fma(-cf[r], u[r][c], xc);
                x[v][c] = xc;
            }
        }
        if (PF && b + 1 < nblk) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < NCW; ++c) u[r][c] = un[PF ? r : 0][PF ? c : 0];
        }
    }
#pragma unroll
    for (int v = 0; v < VPB; ++v)
#pragma unroll
        for (int c = 0; c < NCW; ++c) {
            const int64_t i = i0 + 32 * c;
            if (v0 + v < k && i < w) evecs[i * lde + v0 + v] = x[v][c];
        }
}

__global__ void k_info_init(int32_t* info) {
    info[0] = 1;
    info[1] = 0;
}

}  // namespace

int64_t syev_topk_ws_bytes(int64_t w, int64_t k) {
    // A, Uh (w^2 each), d, e, e2, beta, p (w each), bounds, X (k w), fac (k 5w), clusters
    const int64_t dbl = 2 * w * w + 6 * w + 16 + k * w + 5 * k * w + 1024 + (w / kBtRows + 2) * kBtG;
    return dbl * (int64_t)sizeof(double) + (k + 2) * 4 + 256;
}

int syev_topk(int64_t w, const double* M, int64_t ldm, int64_t k, double* evals, double* evecs, int64_t lde,
              int32_t* info, void* ws, int64_t ws_bytes, cudaStream_t st) {
    RSVD_REQUIRE(w >= 1 && k >= 1 && k <= w, "syev_topk: bad shape");
    RSVD_REQUIRE(ws_bytes >= syev_topk_ws_bytes(w, k), "syev_topk: workspace too small");
    double* base = (double*)ws;
    TriState s;
    s.w = w;
    s.A = base;
    s.Uh = s.A + w * w;
    s.d = s.Uh + w * w;
    s.e = s.d + w;
    double* e2 = s.e + w;
    s.beta = e2 + w;
    s.p = s.beta + w;
    s.p2 = s.p + w;
    double* bounds = s.p2 + w;
    double* X = bounds + 16;
    double* fac = X + k * w;
    s.partial = fac + 5 * k * w;
    s.bar = (unsigned int*)(s.partial + 1024 - 16);
    double* btg = s.partial + 1024;  // (w / kBtRows + 2) x kBtRows^2 block Grams
    int32_t* cl = (int32_t*)(btg + (w / kBtRows + 2) * kBtG);
    int32_t* ncl = cl + k + 1;
    RSVD_CHECK_CUDA(cudaMemsetAsync(s.bar, 0, 2 * sizeof(unsigned int), st));
    k_info_init<<<1, 1, 0, st>>>(info);
    k_copy_sym<<<(unsigned)cdiv(w * w, 256), 256, 0, st>>>(w, M, ldm, s.A);
    RSVD_CHECK_LAUNCH();
    bool done = false;
    if (w <= kClTriMaxW && !getenv("RSVD_TRIDIAG_GRID")) {
        const int nloc = (int)((w + kClTri - 1) / kClTri);
        // one cluster barrier per column unless RSVD_TRIDIAG_TWO_BARRIER (A/B)
        const bool one = w >= 4 && getenv("RSVD_TRIDIAG_TWO_BARRIER") == nullptr;
        const size_t csm = ((size_t)nloc * w + 6 * (size_t)w) * sizeof(double);
        // cluster launch supported and schedulable (checked once per device;
        // slot value 0 = unchecked, 1 = no, 2 = yes)
        static PerDevice<int> cluster_dev;
        int& cluster_slot = cluster_dev.get();
        int cluster_ok = cluster_slot - 1;
        if (cluster_ok < 0) {
            cluster_ok = 0;
            const int maxsm = (int)(((size_t)((kClTriMaxW + kClTri - 1) / kClTri) * kClTriMaxW + 6 * (size_t)kClTriMaxW) *
                                    sizeof(double));
            if (cudaFuncSetAttribute(k_tridiag_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                    cudaSuccess &&
                cudaFuncSetAttribute(k_tridiag_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) ==
                    cudaSuccess &&
                cudaFuncSetAttribute(k_tridiag_cluster1, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                    cudaSuccess &&
                cudaFuncSetAttribute(k_tridiag_cluster1, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) ==
                    cudaSuccess) {
                cudaLaunchConfig_t qc = {};
                qc.gridDim = dim3(kClTri);
                qc.blockDim = dim3(kClTriThreads);
                qc.dynamicSmemBytes = (size_t)maxsm;
                cudaLaunchAttribute qa[1];
                qa[0].id = cudaLaunchAttributeClusterDimension;
                qa[0].val.clusterDim.x = kClTri;
                qa[0].val.clusterDim.y = 1;
                qa[0].val.clusterDim.z = 1;
                qc.attrs = qa;
                qc.numAttrs = 1;
                int nclusters = 0;
                if (cudaOccupancyMaxActiveClusters(&nclusters, k_tridiag_cluster, &qc) == cudaSuccess &&
                    nclusters >= 1)
                    cluster_ok = 1;
            }
            cudaGetLastError();  // clear a refused attribute / query (grid kernel below)
            cluster_slot = cluster_ok + 1;
        }
        if (cluster_ok == 1) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(kClTri);
            cfg.blockDim = dim3(kClTriThreads);
            cfg.dynamicSmemBytes = csm;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = kClTri;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if (one)
                RSVD_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_tridiag_cluster1, s));
            else
                RSVD_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_tridiag_cluster, s));
            done = true;
        }
    }
    if (!done) {
        // one barrier per column (k_tridiag1) unless RSVD_TRIDIAG_TWO_BARRIER is set (A/B);
        // the matrix in distributed shared memory (k_tridiag_sm) when it fits
        const bool two = getenv("RSVD_TRIDIAG_TWO_BARRIER") != nullptr;
        const bool one = w >= 4 && !two;
        const int64_t gsm = sm_count();
        const size_t smsz = ((size_t)cdiv(w, gsm) * w + 4 * w) * sizeof(double);
        const bool dsm = one && w <= 4 * kTriThreads && smsz <= 220 * 1024 && getenv("RSVD_TRIDIAG_L2") == nullptr;
        if (dsm) {
            RSVD_CHECK_CUDA(cudaFuncSetAttribute(k_tridiag_sm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smsz));
            int per = 0;
            RSVD_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tridiag_sm, kTriThreads, smsz));
            RSVD_REQUIRE(per >= 1, "syev_topk: distributed tridiagonalisation cannot be resident");
            void* args[] = {&s};
            RSVD_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)k_tridiag_sm, dim3((unsigned)gsm),
                                                        dim3(kTriThreads), args, smsz, st));
            done = true;
        }
    }
    if (!done) {
        const bool two = getenv("RSVD_TRIDIAG_TWO_BARRIER") != nullptr;
        const bool one = w >= 4 && !two;
        const void* kern = one ? (const void*)k_tridiag1 : (const void*)k_tridiag;
        const size_t smem = (size_t)((one ? 4 : 2) * w) * sizeof(double);
        RSVD_REQUIRE(smem <= 200 * 1024, "syev_topk: w too large");
        if (smem > 48 * 1024)
            RSVD_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        RSVD_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTriThreads, smem));
        RSVD_REQUIRE(per_sm >= 1, "syev_topk: tridiagonalisation kernel cannot be resident");
        // one warp per trailing row at most; the one-barrier kernel's fused
        // pass is latency bound, so it takes every SM (more rows in flight)
        int64_t g = one ? cdiv(w, 8) : cdiv(w, kTriThreads / 32);
        if (g > sm_count()) g = sm_count();
        if (g < 1) g = 1;
        void* args[] = {&s};
        RSVD_CHECK_CUDA(cudaLaunchCooperativeKernel(kern, dim3((unsigned)g), dim3(kTriThreads), args, smem, st));
    }
    k_e2<<<(unsigned)cdiv(w, 256), 256, 0, st>>>(w, s.e, e2);
    RSVD_CHECK_LAUNCH();
    k_tri_bounds<<<1, 1024, 0, st>>>(w, s.d, s.e, bounds);
    RSVD_CHECK_LAUNCH();
    k_multisect<<<(unsigned)cdiv(k * 32, 256), 256, 0, st>>>(w, k, s.d, e2, bounds, evals);
    RSVD_CHECK_LAUNCH();
    if (evecs == nullptr) return RSVD_OK;  // eigenvalues only (the sweep harness's oracle spectrum)
    k_clusters<<<1, 32, 0, st>>>(k, evals, bounds, cl, ncl);
    RSVD_CHECK_LAUNCH();
    k_invit<<<(unsigned)cdiv(k * 32, 128), 128, 0, st>>>(w, k, s.d, s.e, evals, bounds, cl, ncl, X, fac, info);
    RSVD_CHECK_LAUNCH();
    RSVD_REQUIRE(w <= 32 * kBtChunks, "syev_topk: w > %d", 32 * kBtChunks);
    {
        const size_t bsm = (size_t)(2 * kBtRows * ((w + 1) & ~int64_t(1))) * sizeof(double);
        // one vector per CTA below 300 vectors (k = 50: 50 CTAs instead of 7)
        const int vpb = k >= 300 ? 4 : 1;
        const bool seq = getenv("RSVD_BT_SEQ") != nullptr;  // one-by-one reflectors (A/B)
        const bool staged = getenv("RSVD_BT_STAGED") != nullptr;  // smem-staged blocked kernel (A/B)
        if (!seq && w >= 3) {
            const int64_t nblk = (w - 3 + kBtRows) / kBtRows;
            k_bt_gram<<<(unsigned)nblk, 256, 0, st>>>(w, s.Uh, btg);
            RSVD_CHECK_LAUNCH();
        }
        if (!seq && !staged && w >= 3) {
            // row-split kernel: kRsWarps warps x NCW x 32 rows >= w
            const int64_t ncw = cdiv(cdiv(w, kRsWarps), 32);
            auto rs = [&](auto kern, int vp) -> int {
                kern<<<(unsigned)cdiv(k, vp), 32 * kRsWarps, 0, st>>>(w, k, s.Uh, s.beta, btg, X, evecs, lde);
                RSVD_CHECK_LAUNCH();
                return RSVD_OK;
            };
#define RSVD_RS(N)                                                                                     \
            if (ncw <= N) return k >= 64 ? rs(k_backtransform_rs<N, 4>, 4) : rs(k_backtransform_rs<N, 2>, 2);
#define RSVD_RS2(N) \
            if (ncw <= N) return rs(k_backtransform_rs<N, 2>, 2);
            RSVD_RS(1) RSVD_RS(2) RSVD_RS(3) RSVD_RS2(4) RSVD_RS2(5) RSVD_RS2(6) RSVD_RS2(7) RSVD_RS2(8)
#undef RSVD_RS2
#undef RSVD_RS
        }
        auto launch = [&](auto kern, auto kernb, int vp) -> int {
            if (seq || w < 3) {
                if (bsm > 48 * 1024)
                    RSVD_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
                kern<<<(unsigned)cdiv(k, vp), 32 * vp, bsm, st>>>(w, k, s.Uh, s.beta, X, evecs, lde);
            } else {
                if (bsm > 48 * 1024)
                    RSVD_CHECK_CUDA(cudaFuncSetAttribute(kernb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
                kernb<<<(unsigned)cdiv(k, vp), 32 * vp, bsm, st>>>(w, k, s.Uh, s.beta, btg, X, evecs, lde);
            }
            RSVD_CHECK_LAUNCH();
            return RSVD_OK;
        };
#define RSVD_BT(NC)                                                                                    \
        if (w <= 32 * NC)                                                                              \
            return vpb == 1 ? launch(k_backtransform<NC, 1>, k_backtransform_blk<NC, 1>, 1)            \
                            : launch(k_backtransform<NC, 4>, k_backtransform_blk<NC, 4>, 4);
        RSVD_BT(8) RSVD_BT(16) RSVD_BT(20) RSVD_BT(24) RSVD_BT(32) RSVD_BT(40) RSVD_BT(52) RSVD_BT(64)
#undef RSVD_BT
    }
    return RSVD_OK;
}

}  // namespace rsvd
