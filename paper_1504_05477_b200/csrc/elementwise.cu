// Deterministic reductions and element-wise helpers of the path.
#include "common.cuh"

namespace rsvd {

namespace {

constexpr int kColRows = 8;  // rows per block-iteration; 32 columns per block

template <typename T>
__global__ void k_colreduce_partial(int64_t n, int64_t p, const T* __restrict__ X, int64_t ldx,
                                    int square, int64_t rows_per_chunk, double* __restrict__ ws) {
    __shared__ double red[kColRows][33];
    const int lx = threadIdx.x % 32, ly = threadIdx.x / 32;
    const int64_t c = (int64_t)blockIdx.x * 32 + lx;
    const int64_t r0 = (int64_t)blockIdx.y * rows_per_chunk;
    const int64_t r1 = min(n, r0 + rows_per_chunk);
    double acc = 0.0;
    if (c < p) {
        // 8 rows' loads in flight per thread (the chunk is thousands of rows
        // long; one load at a time made this latency bound); the sum is still
        // accumulated in row order
        int64_t r = r0 + ly;
        for (; r + 7 * kColRows < r1; r += 8 * kColRows) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = (double)X[(r + q * kColRows) * ldx + c];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += square ? v[q] * v[q] : v[q];
        }
        for (; r < r1; r += kColRows) {
            double v = (double)X[r * ldx + c];
            acc += square ? v * v : v;
        }
    }
    red[ly][lx] = acc;
    __syncthreads();
    if (ly == 0 && c < p) {
        double s = 0.0;
        for (int i = 0; i < kColRows; ++i) s += red[i][lx];
        ws[(int64_t)blockIdx.y * p + c] = s;
    }
}

// Warp per column: lane l sums partials l, l + 32, ... then a fixed xor tree
// (deterministic; the chunk count is ~600 at p = 50, which one thread per
// column summed serially in ~25 us).
__global__ void k_colreduce_final(int64_t p, int64_t chunks, const double* __restrict__ ws,
                                  double* __restrict__ out) {
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= p) return;
    double s = 0.0;
    for (int64_t i = lane; i < chunks; i += 32) s += ws[i * p + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = s;
}

// (|x|, index) candidate order of the argmax reductions: larger |x| wins, the
// smaller row index on ties (numpy argmax semantics); INT64_MAX marks none.
struct AbsArg {
    double v, x;
    int64_t i;
};

__device__ __forceinline__ void absarg_take(AbsArg& a, double x, int64_t ix) {
    if (ix == INT64_MAX) return;
    const double v = fabs(x);
    if (v > a.v || (v == a.v && ix < a.i)) a = {v, x, ix};
}

__device__ __forceinline__ AbsArg absarg_warp(AbsArg a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        AbsArg b{__shfl_xor_sync(0xffffffffu, a.v, o), __shfl_xor_sync(0xffffffffu, a.x, o),
                 (int64_t)__shfl_xor_sync(0xffffffffu, (long long)a.i, o)};
        if (b.v > a.v || (b.v == a.v && b.i < a.i)) a = b;
    }
    return a;
}

int64_t col_chunks(int64_t n, int64_t p) {
    int64_t target = (int64_t)sm_count() * 8;
    int64_t colblocks = cdiv(p, 32);
    int64_t ch = cdiv(target, colblocks);
    int64_t maxch = cdiv(n, 256);
    if (ch > maxch) ch = maxch;
    if (ch < 1) ch = 1;
    return ch;
}

// argmax |x| per column, first index on ties (numpy argmax semantics).
// Stores the SIGNED value at the argmax so the flip decision never re-reads X.
template <typename T>
__global__ void k_absargmax_partial(int64_t n, int64_t k, const T* __restrict__ X, int64_t ldx,
                                    int64_t rows_per_chunk, double* __restrict__ wv,
                                    int64_t* __restrict__ wi) {
    __shared__ double sv[kColRows][33];
    __shared__ double ss[kColRows][33];
    __shared__ int64_t si[kColRows][33];
    const int lx = threadIdx.x % 32, ly = threadIdx.x / 32;
    const int64_t c = (int64_t)blockIdx.x * 32 + lx;
    const int64_t r0 = (int64_t)blockIdx.y * rows_per_chunk;
    const int64_t r1 = min(n, r0 + rows_per_chunk);
    double best = -1.0, bsig = 0.0;
    int64_t bi = INT64_MAX;
    if (c < k) {
        // rows visited in increasing order (first max kept); 8 loads in flight
        int64_t r = r0 + ly;
        for (; r + 7 * kColRows < r1; r += 8 * kColRows) {
            double xs[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) xs[q] = (double)X[(r + q * kColRows) * ldx + c];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double v = fabs(xs[q]);
                if (v > best) {
                    best = v;
                    bsig = xs[q];
                    bi = r + q * kColRows;
                }
            }
        }
        for (; r < r1; r += kColRows) {
            double x = (double)X[r * ldx + c];
            double v = fabs(x);
            if (v > best) {
                best = v;
                bsig = x;
                bi = r;
            }
        }
    }
    sv[ly][lx] = best;
    ss[ly][lx] = bsig;
    si[ly][lx] = bi;
    __syncthreads();
    if (ly == 0 && c < k) {
        for (int i = 1; i < kColRows; ++i) {
            if (sv[i][lx] > best || (sv[i][lx] == best && si[i][lx] < bi)) {
                best = sv[i][lx];
                bsig = ss[i][lx];
                bi = si[i][lx];
            }
        }
        wv[(int64_t)blockIdx.y * k + c] = bsig;
        wi[(int64_t)blockIdx.y * k + c] = bi;
    }
}

__global__ void k_sign_decide(int64_t k, int64_t chunks, const double* __restrict__ wv,
                              const int64_t* __restrict__ wi, int32_t* __restrict__ flip) {
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= k) return;
    AbsArg a{-1.0, 0.0, INT64_MAX};
    for (int64_t i = lane; i < chunks; i += 32) absarg_take(a, wv[i * k + c], wi[i * k + c]);
    a = absarg_warp(a);
    if (lane == 0) flip[c] = a.x < 0.0;
}

template <typename T>
__global__ void k_sign_flip(int64_t n, int64_t k, T* __restrict__ X, int64_t ldx,
                            const int32_t* __restrict__ flip) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * k) return;
    int64_t r = e / k, c = e % k;
    if (flip[c]) X[r * ldx + c] = -X[r * ldx + c];
}

__global__ void k_absargmax_final(int64_t k, int64_t chunks, const double* __restrict__ wv,
                                  const int64_t* __restrict__ wi, int64_t row_offset,
                                  double* __restrict__ out_val, int64_t* __restrict__ out_idx) {
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= k) return;
    AbsArg a{-1.0, 0.0, INT64_MAX};
    for (int64_t i = lane; i < chunks; i += 32) absarg_take(a, wv[i * k + c], wi[i * k + c]);
    a = absarg_warp(a);
    if (lane == 0) {
        out_val[c] = a.x;
        out_idx[c] = a.i == INT64_MAX ? INT64_MAX : a.i + row_offset;
    }
}

template <typename T>
__global__ void k_flip_by(int64_t n, int64_t k, T* __restrict__ X, int64_t ldx,
                          const double* __restrict__ sign_val) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * k) return;
    int64_t r = e / k, c = e % k;
    if (sign_val[c] < 0.0) X[r * ldx + c] = -X[r * ldx + c];
}

template <typename T>
__global__ void k_mask_cols(int64_t n, int64_t p, T* __restrict__ X, int64_t ldx,
                            const int32_t* __restrict__ keep, const int32_t* __restrict__ pred) {
    if (pred && *pred == 0) return;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * p) return;
    int64_t r = e / p, c = e % p;
    if (!keep[c]) X[r * ldx + c] = T(0);
}

template <typename S, typename D>
__global__ void k_convert(int64_t rows, int64_t cols, const S* __restrict__ src, int64_t lds,
                          D* __restrict__ dst, int64_t ldd, const int32_t* __restrict__ pred) {
    if (pred && *pred == 0) return;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * cols) return;
    int64_t i = e / cols, j = e % cols;
    dst[i * ldd + j] = (D)src[i * lds + j];
}

// dst[i, :] = src[idx[i], :] (GATHER) or dst[idx[i], :] = src[i, :] (scatter):
// the hot-column panels of the hybrid CSR product (sparse.cu).
template <typename T, bool GATHER>
__global__ void k_move_rows(int64_t nidx, int64_t cols, const int64_t* __restrict__ idx, const T* __restrict__ src,
                            int64_t lds, T* __restrict__ dst, int64_t ldd) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nidx * cols) return;
    const int64_t i = e / cols, j = e % cols;
    if (GATHER)
        dst[i * ldd + j] = src[idx[i] * lds + j];
    else
        dst[idx[i] * ldd + j] = src[i * lds + j];
}

__global__ void k_sqrt_clip(int64_t k, const double* __restrict__ in, double* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) out[i] = sqrt(fmax(in[i], 0.0));
}

__global__ void k_ortho_error(int64_t k, const double* __restrict__ G, int64_t ldg,
                              double* __restrict__ out) {
    __shared__ double red[32];
    double m = 0.0;
    for (int64_t e = threadIdx.x; e < k * k; e += blockDim.x) {
        int64_t i = e / k, j = e % k;
        double v = fabs(G[i * ldg + j] - (i == j ? 1.0 : 0.0));
        if (!(v <= m)) m = v;  // NaN propagates
    }
    for (int o = 16; o > 0; o >>= 1) {
        double x = __shfl_xor_sync(0xffffffffu, m, o);
        if (!(x <= m)) m = x;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
            if (!(red[i] <= r)) r = red[i];
        out[0] = r;
    }
}

// Device-side replacement columns from the reference's fixed-seed fill stream
// (factor.py:40, 89-90, 107): SplitMix64 is counter based, so normal j of the
// r-th fill vector (n normals per vector, 2*ceil(n/2) uniforms consumed per
// vector, matrix.py:44-47) is computed directly from its stream position.
// Values equal the host stream up to libm-vs-CUDA last-ulp differences; the
// factorization does not depend on the fill values.
__device__ __forceinline__ uint64_t mix64d(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ULL;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBULL;
    x ^= x >> 31;
    return x;
}

__device__ __forceinline__ double fill_normal(uint64_t seed, int64_t n, int64_t r, int64_t j) {
    const uint64_t g = 0x9E3779B97F4A7C15ULL;
    const uint64_t pair = (uint64_t)r * (uint64_t)((n + 1) / 2) + (uint64_t)(j / 2);
    const uint64_t x1 = mix64d(seed + (2 * pair + 1) * g);
    const uint64_t x2 = mix64d(seed + (2 * pair + 2) * g);
    const double u1 = (double)((x1 >> 11) + 1) * (1.0 / 9007199254740992.0);
    const double u2 = (double)((x2 >> 11) + 1) * (1.0 / 9007199254740992.0);
    const double rad = sqrt(-2.0 * log(u1));
    const double th = 6.283185307179586 * u2;
    return (j & 1) ? rad * sin(th) : rad * cos(th);
}

template <typename T>
__global__ void k_insert_fill(int64_t n, int64_t p, T* __restrict__ X, int64_t ldx,
                              const int32_t* __restrict__ mask, const int32_t* __restrict__ ndef,
                              uint64_t seed, int64_t row_offset, int64_t n_total,
                              const int32_t* __restrict__ pred) {
    extern __shared__ int32_t smask[];
    if (pred && *pred == 0) return;
    if (ndef && ndef[0] == 0) return;
    const int64_t base = ndef ? ndef[1] : 0;
    for (int64_t j = threadIdx.x; j < p; j += blockDim.x) smask[j] = mask[j];
    __syncthreads();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t rank = base;
    for (int64_t j = 0; j < p; ++j) {
        if (smask[j]) {
            X[i * ldx + j] = (T)fill_normal(seed, n_total, rank, row_offset + i);
            ++rank;
        }
    }
}

__global__ void k_fill_stream(int64_t n, int64_t nvec, uint64_t seed, double* __restrict__ out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nvec) return;
    out[e] = fill_normal(seed, n, e / n, e % n);
}

}  // namespace

int64_t colreduce_ws_bytes(int64_t n, int64_t p) {
    return col_chunks(n, p) * p * (int64_t)(sizeof(double) + sizeof(int64_t)) + p * 4 + 256;
}

int colreduce(int dtype, int square, int64_t n, int64_t p, const void* X, int64_t ldx,
              double* out, void* ws, int64_t ws_bytes, cudaStream_t st) {
    if (p == 0) return RSVD_OK;
    int64_t ch = col_chunks(n, p);
    RSVD_REQUIRE(ws_bytes >= ch * p * (int64_t)sizeof(double), "colreduce: workspace too small");
    int64_t rpc = cdiv(n, ch);
    dim3 grid((unsigned)cdiv(p, 32), (unsigned)ch);
    if (dtype == RSVD_F64)
        k_colreduce_partial<double><<<grid, 32 * kColRows, 0, st>>>(n, p, (const double*)X, ldx,
                                                                   square, rpc, (double*)ws);
    else
        k_colreduce_partial<float><<<grid, 32 * kColRows, 0, st>>>(n, p, (const float*)X, ldx,
                                                                  square, rpc, (double*)ws);
    RSVD_CHECK_LAUNCH();
    k_colreduce_final<<<(unsigned)cdiv(p * 32, 256), 256, 0, st>>>(p, ch, (const double*)ws, out);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int canonicalize_signs(int dtype, int64_t n, int64_t k, void* X, int64_t ldx, void* ws,
                       int64_t ws_bytes, cudaStream_t st) {
    if (k == 0 || n == 0) return RSVD_OK;
    int64_t ch = col_chunks(n, k);
    RSVD_REQUIRE(ws_bytes >= ch * k * (int64_t)(sizeof(double) + sizeof(int64_t)) + k * 4,
                 "canonicalize_signs: workspace too small");
    double* wv = (double*)ws;
    int64_t* wi = (int64_t*)(wv + ch * k);
    int32_t* flip = (int32_t*)(wi + ch * k);
    int64_t rpc = cdiv(n, ch);
    dim3 grid((unsigned)cdiv(k, 32), (unsigned)ch);
    unsigned nb = (unsigned)cdiv(n * k, 256);
    if (dtype == RSVD_F64)
        k_absargmax_partial<double><<<grid, 32 * kColRows, 0, st>>>(n, k, (const double*)X, ldx,
                                                                   rpc, wv, wi);
    else
        k_absargmax_partial<float><<<grid, 32 * kColRows, 0, st>>>(n, k, (const float*)X, ldx, rpc,
                                                                  wv, wi);
    RSVD_CHECK_LAUNCH();
    k_sign_decide<<<(unsigned)cdiv(k * 32, 256), 256, 0, st>>>(k, ch, wv, wi, flip);
    RSVD_CHECK_LAUNCH();
    if (dtype == RSVD_F64)
        k_sign_flip<double><<<nb, 256, 0, st>>>(n, k, (double*)X, ldx, flip);
    else
        k_sign_flip<float><<<nb, 256, 0, st>>>(n, k, (float*)X, ldx, flip);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int col_absargmax(int dtype, int64_t n, int64_t k, const void* X, int64_t ldx, int64_t row_offset,
                  double* out_val, int64_t* out_idx, void* ws, int64_t ws_bytes, cudaStream_t st) {
    if (k == 0) return RSVD_OK;
    int64_t ch = col_chunks(n > 0 ? n : 1, k);
    RSVD_REQUIRE(ws_bytes >= ch * k * (int64_t)(sizeof(double) + sizeof(int64_t)),
                 "col_absargmax: workspace too small");
    double* wv = (double*)ws;
    int64_t* wi = (int64_t*)(wv + ch * k);
    int64_t rpc = cdiv(n > 0 ? n : 1, ch);
    dim3 grid((unsigned)cdiv(k, 32), (unsigned)ch);
    if (dtype == RSVD_F64)
        k_absargmax_partial<double><<<grid, 32 * kColRows, 0, st>>>(n, k, (const double*)X, ldx,
                                                                   rpc, wv, wi);
    else
        k_absargmax_partial<float><<<grid, 32 * kColRows, 0, st>>>(n, k, (const float*)X, ldx, rpc,
                                                                  wv, wi);
    RSVD_CHECK_LAUNCH();
    k_absargmax_final<<<(unsigned)cdiv(k * 32, 256), 256, 0, st>>>(k, ch, wv, wi, row_offset, out_val,
                                                              out_idx);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int flip_by_sign(int dtype, int64_t n, int64_t k, void* X, int64_t ldx, const double* sign_val,
                 cudaStream_t st) {
    if (n * k == 0) return RSVD_OK;
    unsigned nb = (unsigned)cdiv(n * k, 256);
    if (dtype == RSVD_F64)
        k_flip_by<double><<<nb, 256, 0, st>>>(n, k, (double*)X, ldx, sign_val);
    else
        k_flip_by<float><<<nb, 256, 0, st>>>(n, k, (float*)X, ldx, sign_val);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int mask_cols(int dtype, int64_t n, int64_t p, void* X, int64_t ldx, const int32_t* keep,
              const int32_t* pred, cudaStream_t st) {
    if (n * p == 0) return RSVD_OK;
    unsigned nb = (unsigned)cdiv(n * p, 256);
    if (dtype == RSVD_F64)
        k_mask_cols<double><<<nb, 256, 0, st>>>(n, p, (double*)X, ldx, keep, pred);
    else
        k_mask_cols<float><<<nb, 256, 0, st>>>(n, p, (float*)X, ldx, keep, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int convert(int sd, int dd, int64_t rows, int64_t cols, const void* src, int64_t lds, void* dst,
            int64_t ldd, const int32_t* pred, cudaStream_t st) {
    if (rows * cols == 0) return RSVD_OK;
    unsigned nb = (unsigned)cdiv(rows * cols, 256);
    if (sd == RSVD_F64 && dd == RSVD_F32)
        k_convert<double, float><<<nb, 256, 0, st>>>(rows, cols, (const double*)src, lds, (float*)dst, ldd, pred);
    else if (sd == RSVD_F32 && dd == RSVD_F64)
        k_convert<float, double><<<nb, 256, 0, st>>>(rows, cols, (const float*)src, lds, (double*)dst, ldd, pred);
    else if (sd == RSVD_F64)
        k_convert<double, double><<<nb, 256, 0, st>>>(rows, cols, (const double*)src, lds, (double*)dst, ldd, pred);
    else
        k_convert<float, float><<<nb, 256, 0, st>>>(rows, cols, (const float*)src, lds, (float*)dst, ldd, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int move_rows(int dtype, int gather, int64_t nidx, int64_t cols, const int64_t* idx, const void* src, int64_t lds,
              void* dst, int64_t ldd, cudaStream_t st) {
    if (nidx == 0 || cols == 0) return RSVD_OK;
    const unsigned nb = (unsigned)cdiv(nidx * cols, 256);
#define RSVD_MR(T, G) k_move_rows<T, G><<<nb, 256, 0, st>>>(nidx, cols, idx, (const T*)src, lds, (T*)dst, ldd)
    if (dtype == RSVD_F64) {
        if (gather) RSVD_MR(double, true); else RSVD_MR(double, false);
    } else {
        if (gather) RSVD_MR(float, true); else RSVD_MR(float, false);
    }
#undef RSVD_MR
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int sqrt_clip(int64_t k, const double* in, double* out, cudaStream_t st) {
    if (k == 0) return RSVD_OK;
    k_sqrt_clip<<<(unsigned)cdiv(k, 256), 256, 0, st>>>(k, in, out);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int ortho_error(int64_t k, const double* G, int64_t ldg, double* out, cudaStream_t st) {
    k_ortho_error<<<1, 1024, 0, st>>>(k, G, ldg, out);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int insert_fill(int dtype, int64_t n, int64_t p, void* X, int64_t ldx, const int32_t* mask,
                const int32_t* ndef, uint64_t seed, int64_t row_offset, int64_t n_total,
                const int32_t* pred, cudaStream_t st) {
    if (n == 0 || p == 0) return RSVD_OK;
    size_t sm = (size_t)p * sizeof(int32_t);
    RSVD_REQUIRE(sm <= 48 * 1024, "insert_fill: p too large");
    unsigned nb = (unsigned)cdiv(n, 256);
    if (dtype == RSVD_F64)
        k_insert_fill<double><<<nb, 256, sm, st>>>(n, p, (double*)X, ldx, mask, ndef, seed,
                                                   row_offset, n_total, pred);
    else
        k_insert_fill<float><<<nb, 256, sm, st>>>(n, p, (float*)X, ldx, mask, ndef, seed,
                                                  row_offset, n_total, pred);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

int fill_stream(int64_t n, int64_t nvec, uint64_t seed, double* out, cudaStream_t st) {
    if (n * nvec == 0) return RSVD_OK;
    k_fill_stream<<<(unsigned)cdiv(n * nvec, 256), 256, 0, st>>>(n, nvec, seed, out);
    RSVD_CHECK_LAUNCH();
    return RSVD_OK;
}

}  // namespace rsvd
