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
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* gen = bar + 1;
        unsigned int g = *gen;
        __threadfence();
        unsigned int arrived = atomicAdd(bar, 1u);
        if (arrived == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) {
                __nanosleep(32);
            }
        }
        __threadfence();
    }
    __syncthreads();
}

}  // namespace rsvd
