// Shared helpers for the sm_100a kernels of the randomized block-Krylov path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/rsvd_b200.h"

namespace rsvd {

void set_error(const char* fmt, ...);

#define RSVD_CHECK_CUDA(expr)                                                     \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) {                                                  \
            ::rsvd::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,          \
                              cudaGetErrorString(_e));                            \
            return RSVD_ERR_CUDA;                                                 \
        }                                                                         \
    } while (0)

#define RSVD_CHECK_LAUNCH() RSVD_CHECK_CUDA(cudaGetLastError())

#define RSVD_REQUIRE(cond, ...)                                                   \
    do {                                                                          \
        if (!(cond)) {                                                            \
            ::rsvd::set_error(__VA_ARGS__);                                       \
            return RSVD_ERR_INVALID;                                              \
        }                                                                         \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();
int current_device();  // cudaGetDevice, clamped to [0, kMaxDevices)

// Process state keyed by the calling thread's current CUDA device: the
// once-per-device cudaFuncSetAttribute flags and the grow-only scratch
// buffers. A process that drives several GPUs gets a separate slot per
// device (kernel attributes are per device; a scratch pointer of one device
// must never reach another device's kernels).
constexpr int kMaxDevices = 64;
template <typename T>
struct PerDevice {
    T slot[kMaxDevices]{};
    T& get() { return slot[current_device()]; }
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sense-reversing grid barrier for cooperative launches (all CTAs resident).
// bar[0] = arrival count (must start at 0), bar[1] = generation.
// Grid-wide barrier of a cooperative launch (bar[0] zeroed before the launch):
// ONE atomic per CTA on a counter that only grows -- arrival number `old`
// belongs to generation old / nblocks, which ends when the counter reaches the
// next multiple of nblocks -- and a spin on that counter. (The first version
// reset the counter and bumped a separate generation word: two more dependent
// L2 round trips per barrier by the last arriver, ~1 us of the ~7 us a column
// of the grid tridiagonalisation takes.)
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int old = atomicAdd(bar, 1u);
        const unsigned int target = (old / nblocks + 1u) * nblocks;
        volatile unsigned int* cnt = bar;
        while ((int)(*cnt - target) < 0) {
        }
        __threadfence();
    }
    __syncthreads();
}

}  // namespace rsvd
