// tcgen05 3xTF32 tall-skinny GEMM (placeholder until the kernel lands).
#include "gemm.cuh"

namespace rsvd {

bool gemm_tc_nn_supported(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, const void*,
                          const void*) {
    return false;
}
int gemm_nn_tc(int64_t, int64_t, int64_t, double, const float*, int64_t, const float*, int64_t,
               double, float*, int64_t, const double*, cudaStream_t) {
    set_error("gemm_nn_tc: not built");
    return RSVD_ERR_INVALID;
}
bool gemm_tc_tn_supported(int64_t, int64_t, int64_t, int64_t, int64_t, const void*, const void*) {
    return false;
}
int64_t gemm_tn_tc_ws_bytes(int64_t, int64_t, int64_t) { return 0; }
int gemm_tn_tc(int, int64_t, int64_t, int64_t, double, const float*, int64_t, const float*,
               int64_t, double, void*, int64_t, const double*, const double*, void*, int64_t,
               cudaStream_t) {
    set_error("gemm_tn_tc: not built");
    return RSVD_ERR_INVALID;
}

}  // namespace rsvd
