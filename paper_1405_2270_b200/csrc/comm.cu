// comm.cu -- the one collective of the sharded path: NCCL all-reduce of functional partials.
//
// the N^3 expansion shards into contiguous z-slab ranges with no exchange (the
// reference's k-slab parallel_for, canonical.hpp:251-266, across GPUs instead of threads);
// every rank recomputes the (microsecond) generator and assembly, and the only inter-GPU
// traffic is the all-reduce of the energy / functional partial sums. This file gives the C ABI
// a communicator for that: one process per GPU, ranks joined through an ncclUniqueId that the
// caller moves between processes (a file, a socket, an MPI broadcast, torch.distributed ...).
//
// NCCL is loaded with dlopen on first use instead of being a link dependency: a process that
// never builds a communicator does not need it, and one that already loaded libnccl.so.2 (for
// instance through torch) shares that copy instead of mixing two NCCL builds.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

struct ls_comm {
    ncclComm_t comm = nullptr;
    int world = 0;
    int rank = 0;
    int device = -1;
};

namespace {

struct Nccl {
    void* handle = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string load_error;
};

const Nccl& nccl() {
    static Nccl lib;
    static std::once_flag once;
    std::call_once(once, [] {
        lib.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib.handle) {
            const char* e = dlerror();
            lib.load_error = std::string("dlopen libnccl.so.2: ") + (e ? e : "unknown error");
            return;
        }
        auto sym = [&](const char* name) { return dlsym(lib.handle, name); };
        lib.get_unique_id = reinterpret_cast<decltype(lib.get_unique_id)>(sym("ncclGetUniqueId"));
        lib.comm_init_rank = reinterpret_cast<decltype(lib.comm_init_rank)>(sym("ncclCommInitRank"));
        lib.comm_destroy = reinterpret_cast<decltype(lib.comm_destroy)>(sym("ncclCommDestroy"));
        lib.all_reduce = reinterpret_cast<decltype(lib.all_reduce)>(sym("ncclAllReduce"));
        lib.error_string = reinterpret_cast<decltype(lib.error_string)>(sym("ncclGetErrorString"));
        if (!lib.get_unique_id || !lib.comm_init_rank || !lib.comm_destroy || !lib.all_reduce || !lib.error_string)
            lib.load_error = "libnccl.so.2 lacks an expected symbol";
    });
    return lib;
}

int nccl_ready() {
    const Nccl& n = nccl();
    if (!n.load_error.empty()) return ls::fail(LS_ECUDA, n.load_error);
    return LS_OK;
}

int nccl_fail(ncclResult_t r, const char* where) {
    return ls::fail(LS_ECUDA, std::string(where) + ": " + nccl().error_string(r));
}

}  // namespace

extern "C" {

int ls_comm_unique_id(void* id_out, int bytes) {
    if (!id_out || bytes < static_cast<int>(sizeof(ncclUniqueId)))
        return ls::fail(LS_EVALIDATION, "comm_unique_id: need a buffer of LS_COMM_ID_BYTES bytes");
    if (const int rc = nccl_ready()) return rc;
    ncclUniqueId id;
    if (const ncclResult_t r = nccl().get_unique_id(&id)) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
    return LS_OK;
}

int ls_comm_init(int world, int rank, const void* id, int bytes, ls_comm** out) {
    if (!out) return ls::fail(LS_EVALIDATION, "comm_init: null output");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return ls::fail(LS_EVALIDATION, "comm_init: bad rank / world");
    if (!id || bytes < static_cast<int>(sizeof(ncclUniqueId)))
        return ls::fail(LS_EVALIDATION, "comm_init: need the LS_COMM_ID_BYTES-byte id of rank 0");
    if (const int rc = nccl_ready()) return rc;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ls_comm* c = new ls_comm;
    c->world = world;
    c->rank = rank;
    if (cudaGetDevice(&c->device) != cudaSuccess) {
        delete c;
        return ls::fail(LS_ECUDA, "comm_init: no CUDA device");
    }
    if (const ncclResult_t r = nccl().comm_init_rank(&c->comm, world, uid, rank)) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *out = c;
    return LS_OK;
}

int ls_comm_destroy(ls_comm* c) {
    if (!c) return LS_OK;
    int rc = LS_OK;
    if (c->comm) {
        ls::DeviceGuard g(c->device);
        if (const ncclResult_t r = nccl().comm_destroy(c->comm)) rc = nccl_fail(r, "ncclCommDestroy");
    }
    delete c;
    return rc;
}

int ls_comm_info(const ls_comm* c, int* world, int* rank) {
    if (!c) return ls::fail(LS_EVALIDATION, "comm_info: null communicator");
    if (world) *world = c->world;
    if (rank) *rank = c->rank;
    return LS_OK;
}

int ls_comm_allreduce_f64(ls_comm* c, double* buf_d, int64_t n, int op, void* stream) {
    if (!c) return ls::fail(LS_EVALIDATION, "comm_allreduce: null communicator");
    if (n < 0) return ls::fail(LS_EVALIDATION, "comm_allreduce: negative count");
    if (op != LS_REDUCE_SUM && op != LS_REDUCE_MAX) return ls::fail(LS_EVALIDATION, "comm_allreduce: unknown op");
    if (n == 0) return LS_OK;
    ls::DeviceGuard g(c->device);
    const ncclResult_t r = nccl().all_reduce(buf_d, buf_d, static_cast<size_t>(n), ncclFloat64,
                                             op == LS_REDUCE_SUM ? ncclSum : ncclMax, c->comm,
                                             ls::as_stream(stream));
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
    return LS_OK;
}

int ls_pipeline_energy_allreduce(ls_pipeline* p, const double* r1_d, const double* r2_d, const double* r3_d,
                                 int64_t k0, int64_t k1, double* out_d, ls_comm* c, void* stream) {
    if (const int rc = ls_pipeline_energy(p, r1_d, r2_d, r3_d, k0, k1, out_d, stream)) return rc;
    return ls_comm_allreduce_f64(c, out_d, 1, LS_REDUCE_SUM, stream);
}

}  // extern "C"
