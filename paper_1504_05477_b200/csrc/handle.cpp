// Per-device handle and communicator injection for the C ABI (SURVEY 8(b):
// "an opaque per-device handle that is thread-compatible, not thread-safe"
// and "NCCL communicator injection").
//
// The row-sharded factorization needs one collective: an
// in-place sum-allreduce of the d x p / p x p partials of every reduction over
// rows. A caller that drives the kernels through the C ABI (rather than the
// Python package, which uses torch.distributed) hands the library either an
// existing ncclComm_t (rsvd_handle_set_comm) or a NCCL unique id to build one
// (rsvd_nccl_unique_id + rsvd_handle_init_comm); rsvd_handle_allreduce_sum is
// then stream-ordered with the kernels. NCCL is resolved at run time
// (dlopen("libnccl.so.2"): the copy a host framework has already loaded, else
// the system one), so the library has no link-time NCCL dependency and a
// single-GPU user never loads it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

#include <new>

#include "../../include/rsvd_b200.h"

namespace rsvd {
void set_error(const char* fmt, ...);
}

namespace {

typedef int nccl_result_t;  // ncclResult_t (0 = ncclSuccess)
typedef void* nccl_comm_t;  // ncclComm_t
struct nccl_unique_id_t {
    char internal[128];
};
typedef nccl_result_t (*fn_get_unique_id)(nccl_unique_id_t*);
typedef nccl_result_t (*fn_comm_init_rank)(nccl_comm_t*, int, nccl_unique_id_t, int);
typedef nccl_result_t (*fn_comm_destroy)(nccl_comm_t);
typedef nccl_result_t (*fn_all_reduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t);
typedef const char* (*fn_error_string)(nccl_result_t);

struct NcclApi {
    bool tried = false, ok = false;
    fn_get_unique_id get_unique_id = nullptr;
    fn_comm_init_rank comm_init_rank = nullptr;
    fn_comm_destroy comm_destroy = nullptr;
    fn_all_reduce all_reduce = nullptr;
    fn_error_string error_string = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.tried) {
        api.tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.get_unique_id = (fn_get_unique_id)dlsym(h, "ncclGetUniqueId");
            api.comm_init_rank = (fn_comm_init_rank)dlsym(h, "ncclCommInitRank");
            api.comm_destroy = (fn_comm_destroy)dlsym(h, "ncclCommDestroy");
            api.all_reduce = (fn_all_reduce)dlsym(h, "ncclAllReduce");
            api.error_string = (fn_error_string)dlsym(h, "ncclGetErrorString");
            api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce;
        }
    }
    return api;
}

const char* nccl_err(nccl_result_t r) {
    NcclApi& a = nccl();
    return a.error_string ? a.error_string(r) : "unknown NCCL error";
}

// ncclDataType_t / ncclRedOp_t values used here (nccl.h)
constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0;

}  // namespace

struct rsvd_handle_s {
    int device = 0;
    int world = 1, rank = 0;
    nccl_comm_t comm = nullptr;
    bool owns_comm = false;  // created by rsvd_handle_init_comm (destroyed with the handle)
};

extern "C" {

int rsvd_handle_create(int device, rsvd_handle* out) {
    if (!out) {
        rsvd::set_error("handle_create: null output");
        return RSVD_ERR_INVALID;
    }
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        rsvd::set_error("handle_create: no CUDA device %d", device);
        return RSVD_ERR_CUDA;
    }
    rsvd_handle h = new (std::nothrow) rsvd_handle_s;
    if (!h) {
        rsvd::set_error("handle_create: out of host memory");
        return RSVD_ERR_CUDA;
    }
    h->device = device;
    *out = h;
    return RSVD_OK;
}

int rsvd_handle_destroy(rsvd_handle h) {
    if (!h) return RSVD_OK;
    if (h->owns_comm && h->comm && nccl().ok) nccl().comm_destroy(h->comm);
    delete h;
    return RSVD_OK;
}

int rsvd_handle_device(rsvd_handle h, int* device) {
    if (!h || !device) {
        rsvd::set_error("handle_device: null argument");
        return RSVD_ERR_INVALID;
    }
    *device = h->device;
    return RSVD_OK;
}

int rsvd_handle_world(rsvd_handle h, int* world, int* rank) {
    if (!h || !world || !rank) {
        rsvd::set_error("handle_world: null argument");
        return RSVD_ERR_INVALID;
    }
    *world = h->world;
    *rank = h->rank;
    return RSVD_OK;
}

int rsvd_handle_set_comm(rsvd_handle h, void* nccl_comm, int world, int rank) {
    if (!h || world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_comm)) {
        rsvd::set_error("handle_set_comm: invalid communicator (world %d, rank %d)", world, rank);
        return RSVD_ERR_INVALID;
    }
    if (world > 1 && !nccl().ok) {
        rsvd::set_error("handle_set_comm: libnccl.so.2 could not be loaded");
        return RSVD_ERR_CUDA;
    }
    if (h->owns_comm && h->comm) nccl().comm_destroy(h->comm);
    h->comm = nccl_comm;
    h->owns_comm = false;
    h->world = world;
    h->rank = rank;
    return RSVD_OK;
}

int rsvd_nccl_unique_id(char* id_out, int64_t id_bytes) {
    if (!id_out || id_bytes < 128) {
        rsvd::set_error("nccl_unique_id: need a 128-byte buffer");
        return RSVD_ERR_INVALID;
    }
    if (!nccl().ok) {
        rsvd::set_error("nccl_unique_id: libnccl.so.2 could not be loaded");
        return RSVD_ERR_CUDA;
    }
    nccl_unique_id_t id;
    const nccl_result_t r = nccl().get_unique_id(&id);
    if (r != 0) {
        rsvd::set_error("ncclGetUniqueId: %s", nccl_err(r));
        return RSVD_ERR_CUDA;
    }
    memcpy(id_out, id.internal, 128);
    return RSVD_OK;
}

int rsvd_handle_init_comm(rsvd_handle h, const char* id, int64_t id_bytes, int world, int rank) {
    if (!h || !id || id_bytes < 128 || world < 1 || rank < 0 || rank >= world) {
        rsvd::set_error("handle_init_comm: invalid arguments");
        return RSVD_ERR_INVALID;
    }
    if (!nccl().ok) {
        rsvd::set_error("handle_init_comm: libnccl.so.2 could not be loaded");
        return RSVD_ERR_CUDA;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(h->device) != cudaSuccess) {
        cudaGetLastError();
        rsvd::set_error("handle_init_comm: cannot select device %d", h->device);
        return RSVD_ERR_CUDA;
    }
    nccl_unique_id_t uid;
    memcpy(uid.internal, id, 128);
    nccl_comm_t comm = nullptr;
    const nccl_result_t r = nccl().comm_init_rank(&comm, world, uid, rank);
    cudaSetDevice(prev);
    if (r != 0) {
        rsvd::set_error("ncclCommInitRank: %s", nccl_err(r));
        return RSVD_ERR_CUDA;
    }
    if (h->owns_comm && h->comm) nccl().comm_destroy(h->comm);
    h->comm = comm;
    h->owns_comm = true;
    h->world = world;
    h->rank = rank;
    return RSVD_OK;
}

int rsvd_handle_allreduce_sum(rsvd_handle h, void* buf, int64_t count, int dtype, void* stream) {
    if (!h || count < 0 || (count > 0 && !buf) || (dtype != RSVD_F32 && dtype != RSVD_F64)) {
        rsvd::set_error("handle_allreduce_sum: invalid arguments");
        return RSVD_ERR_INVALID;
    }
    if (!h->comm || count == 0) return RSVD_OK;  // no communicator: one rank, the partial sum is the sum
    const nccl_result_t r =
        nccl().all_reduce(buf, buf, (size_t)count, dtype == RSVD_F64 ? kNcclFloat64 : kNcclFloat32, kNcclSum, h->comm,
                          reinterpret_cast<cudaStream_t>(stream));
    if (r != 0) {
        rsvd::set_error("ncclAllReduce: %s", nccl_err(r));
        return RSVD_ERR_CUDA;
    }
    return RSVD_OK;
}

}  // extern "C"
