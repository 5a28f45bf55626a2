// Device-predicated sections as CUDA-graph conditional (IF) nodes.
//
// The orthonormalization's rarely-taken branches (round 2 of the deflation
// test, the collapsed-fill repair; factor.py:105-116) are decided on the
// device, so a captured factorization holds them as kernels that check a
// device flag and exit. Each such launch still costs ~2 us of graph
// execution (C2: 284 of 756 launches; C1: 394 of 930). Under stream capture,
// rsvd_cond_begin turns the section into an IF node whose condition a
// one-thread kernel sets from the flag, and routes the section's launches
// into the node's body graph; outside capture it is a no-op and the section
// runs eagerly with its per-kernel predicates (which stay in place either
// way, so both paths compute the same thing).
#include "common.cuh"

namespace rsvd {
namespace {

__global__ void k_set_cond(cudaGraphConditionalHandle h, const int32_t* __restrict__ flag) {
    cudaGraphSetConditional(h, (flag && *flag != 0) ? 1u : 0u);
}

}  // namespace
}  // namespace rsvd

using namespace rsvd;

extern "C" {

int rsvd_cond_begin(void* stream, const int32_t* flag, void* body_stream, int32_t* opened) {
    RSVD_REQUIRE(opened != nullptr && body_stream != nullptr && body_stream != stream,
                 "cond_begin: need a separate body stream and an output flag");
    *opened = 0;
    cudaStream_t st = as_stream(stream), bs = as_stream(body_stream);
    cudaStreamCaptureStatus status;
    RSVD_CHECK_CUDA(cudaStreamIsCapturing(st, &status));
    if (status != cudaStreamCaptureStatusActive) return RSVD_OK;  // eager: caller runs the section inline

    cudaGraph_t graph = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    unsigned long long id = 0;
    RSVD_CHECK_CUDA(cudaStreamGetCaptureInfo(st, &status, &id, &graph, &deps, &ndeps));
    cudaGraphConditionalHandle h;
    RSVD_CHECK_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault));
    k_set_cond<<<1, 1, 0, st>>>(h, flag);
    RSVD_CHECK_LAUNCH();
    RSVD_CHECK_CUDA(cudaStreamGetCaptureInfo(st, &status, &id, &graph, &deps, &ndeps));

    cudaGraphNodeParams params = {};
    params.type = cudaGraphNodeTypeConditional;
    params.conditional.handle = h;
    params.conditional.type = cudaGraphCondTypeIf;
    params.conditional.size = 1;
    cudaGraphNode_t node;
    RSVD_CHECK_CUDA(cudaGraphAddNode(&node, graph, deps, ndeps, &params));
    cudaGraph_t body = params.conditional.phGraph_out[0];
    // later work on the capturing stream runs after the conditional node
    RSVD_CHECK_CUDA(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    RSVD_CHECK_CUDA(cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    *opened = 1;
    return RSVD_OK;
}

int rsvd_cond_end(void* body_stream) {
    cudaGraph_t g = nullptr;
    RSVD_CHECK_CUDA(cudaStreamEndCapture(as_stream(body_stream), &g));
    return RSVD_OK;
}

}  // extern "C"
