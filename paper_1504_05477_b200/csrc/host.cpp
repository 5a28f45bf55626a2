// Host-side part of the C ABI: error channel, device queries, and the
// SplitMix64 + Box-Muller Gaussian stream (rsvd_gauss_fill).
//
// The stream must be bit-identical to the reference (_kernels.pyx:22-53),
// whose extension is built with -ffp-contract=off -fno-builtin-sin
// -fno-builtin-cos (pkg/setup.py:15-19); this file is compiled with the same
// flags by the package build, and calls glibc's scalar log/sqrt/cos/sin.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/rsvd_b200.h"

namespace rsvd {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
    return dev;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cached[dev] = n;
    }
    return cached[dev];
}

static inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ULL;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBULL;
    x ^= x >> 31;
    return x;
}

}  // namespace rsvd

extern "C" {

const char* rsvd_last_error(void) { return rsvd::g_err; }

int rsvd_abi_version(void) { return 1; }

int rsvd_sm_count(void) { return rsvd::sm_count(); }

int rsvd_gauss_fill(int64_t count, uint64_t state, double* out, uint64_t* new_state) {
    if (count < 0 || (count > 0 && !out)) {
        rsvd::set_error("gauss_fill: invalid count/output");
        return RSVD_ERR_INVALID;
    }
    const uint64_t inc = 0x9E3779B97F4A7C15ULL;
    const double scale = 1.0 / 9007199254740992.0;  // 2^-53
    const double tau = 6.283185307179586;
    uint64_t s = state;
    int64_t i = 0;
    while (i < count) {
        s += inc;
        const uint64_t x1 = rsvd::mix64(s);
        s += inc;
        const uint64_t x2 = rsvd::mix64(s);
        const double u1 = (double)((x1 >> 11) + 1) * scale;
        const double u2 = (double)((x2 >> 11) + 1) * scale;
        const double radius = sqrt(-2.0 * log(u1));
        const double theta = tau * u2;
        out[i] = radius * cos(theta);
        if (++i < count) out[i++] = radius * sin(theta);
    }
    if (new_state) *new_state = s;
    return RSVD_OK;
}

}  // extern "C"
