// CSR products: spmm_nt (_kernels.pyx:74-92) and, on the CSR of A^T built
// once per operator, spmm_t (_kernels.pyx:95-113) as a deterministic gather
// (no atomics). Warp per row: the warp loads 32 (col, val) pairs at a time,
// broadcasts each with a shuffle, and every lane accumulates NPL contiguous
// columns of the dense row B[col, :] (coalesced 32*NPL-wide reads).
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
