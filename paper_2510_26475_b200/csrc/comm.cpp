// comm.cpp -- the rollout path's one collective: the drafter-gradient
// all-reduce of the prompt-sharded KD update, NCCL over NVLink / NVSwitch, owned by the library
// so the host side needs no PyTorch.
//
// Reference: the gradient of kd_update is a plain sum over the selected samples
// (learner.cpp:68-80); with prompt sharding each rank sums its own samples and the ranks' sums
// are added here. Sharded generation itself needs no collective (server.cpp:266-349 runs one
// engine per request set).
//
// NCCL is bound at run time (dlopen of libnccl.so.2): a process that already loaded NCCL (e.g.
// through PyTorch) shares that copy, and the library itself has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "abi.h"
#include "common.cuh"
#include "engine.h"

namespace {
using rs_abi::guard;
using rs_abi::need;

struct NcclApi {
    decltype(&ncclGetVersion) version = nullptr;
    decltype(&ncclGetUniqueId) unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string load_error;
};

const NcclApi &nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char *e = dlerror();
            a.load_error = std::string("NCCL not loadable: ") + (e ? e : "libnccl.so.2 not found");
            return a;
        }
        a.version = reinterpret_cast<decltype(a.version)>(dlsym(h, "ncclGetVersion"));
        a.unique_id = reinterpret_cast<decltype(a.unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.version || !a.unique_id || !a.init_rank || !a.destroy || !a.all_reduce || !a.error_string)
            a.load_error = "NCCL: missing symbols in libnccl.so.2";
        return a;
    }();
    if (!api.load_error.empty()) throw std::runtime_error(api.load_error);
    return api;
}

void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct rs_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
    rs::DBuf<double> scratch;  // small host all-reduces (losses, timings, token counts)
    std::mutex mu;
    ~rs_comm() {
        if (comm) nccl().destroy(comm);
    }
};

extern "C" {

int rs_nccl_version(int32_t *out) {
    return guard([&] {
        need(out, "rs_nccl_version: out");
        int v = 0;
        nccl_check(nccl().version(&v), "ncclGetVersion");
        *out = v;
    });
}

int rs_comm_unique_id(uint8_t *id) {
    return guard([&] {
        need(id, "rs_comm_unique_id: id");
        static_assert(sizeof(ncclUniqueId) == RS_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        nccl_check(nccl().unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int rs_comm_create(rs_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t *id, rs_comm **out) {
    return guard([&] {
        need(ctx, "rs_comm_create");
        need(id, "rs_comm_create: id");
        need(out, "rs_comm_create: out");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("rs_comm_create: bad rank / nranks");
        RS_CUDA(cudaSetDevice(ctx->device));
        auto c = std::make_unique<rs_comm>();
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        nccl_check(nccl().init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
        c->nranks = nranks;
        c->rank = rank;
        c->device = ctx->device;
        c->scratch.alloc(64);
        *out = c.release();
    });
}

int rs_comm_destroy(rs_comm *c) {
    return guard([&] { delete c; });
}

int rs_comm_size(const rs_comm *c, int32_t *nranks, int32_t *rank) {
    return guard([&] {
        need(c, "rs_comm_size");
        if (nranks) *nranks = c->nranks;
        if (rank) *rank = c->rank;
    });
}

// In-place all-reduce of a device buffer, enqueued on the context's stream.
int rs_comm_allreduce(rs_comm *c, rs_ctx *ctx, void *buf_dev, int64_t count, int32_t dtype, int32_t op) {
    return guard([&] {
        need(c, "rs_comm_allreduce");
        need(ctx, "rs_comm_allreduce: ctx");
        if (count < 0) throw std::invalid_argument("rs_comm_allreduce: negative count");
        if (count == 0) return;
        need(buf_dev, "rs_comm_allreduce: buffer");
        if (ctx->device != c->device) throw std::invalid_argument("rs_comm_allreduce: context on another device");
        const ncclDataType_t t = dtype == RS_DT_F32 ? ncclFloat32 : dtype == RS_DT_F64 ? ncclFloat64 :
                                 dtype == RS_DT_I64 ? ncclInt64 : throw std::invalid_argument("rs_comm_allreduce: dtype");
        const ncclRedOp_t o = op == RS_OP_SUM ? ncclSum : op == RS_OP_MAX ? ncclMax :
                              throw std::invalid_argument("rs_comm_allreduce: op");
        std::lock_guard<std::mutex> lk(c->mu);
        nccl_check(nccl().all_reduce(buf_dev, buf_dev, (size_t)count, t, o, c->comm, ctx->stream), "ncclAllReduce");
    });
}

// All-reduce of a few host doubles (synchronous): losses, token counts, max-over-ranks times.
int rs_comm_allreduce_host(rs_comm *c, rs_ctx *ctx, double *vals, int32_t n, int32_t op) {
    return guard([&] {
        need(c, "rs_comm_allreduce_host");
        need(ctx, "rs_comm_allreduce_host: ctx");
        if (n < 0 || n > 64) throw std::invalid_argument("rs_comm_allreduce_host: 0..64 values");
        if (n == 0) return;
        need(vals, "rs_comm_allreduce_host: values");
        const ncclRedOp_t o = op == RS_OP_SUM ? ncclSum : op == RS_OP_MAX ? ncclMax :
                              throw std::invalid_argument("rs_comm_allreduce_host: op");
        std::lock_guard<std::mutex> lk(c->mu);
        RS_CUDA(cudaMemcpyAsync(c->scratch.p, vals, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        nccl_check(nccl().all_reduce(c->scratch.p, c->scratch.p, (size_t)n, ncclFloat64, o, c->comm, ctx->stream),
                   "ncclAllReduce");
        RS_CUDA(cudaMemcpyAsync(vals, c->scratch.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        RS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// Device memory owned by the library (gradient buffers without a tensor framework).
int rs_device_alloc(rs_ctx *ctx, int64_t bytes, void **out) {
    return guard([&] {
        need(ctx, "rs_device_alloc");
        need(out, "rs_device_alloc: out");
        if (bytes < 0) throw std::invalid_argument("rs_device_alloc: negative size");
        RS_CUDA(cudaSetDevice(ctx->device));
        void *p = nullptr;
        if (bytes) RS_CUDA(cudaMalloc(&p, (size_t)bytes));
        *out = p;
    });
}
int rs_device_free(rs_ctx *ctx, void *p) {
    return guard([&] {
        need(ctx, "rs_device_free");
        if (p) RS_CUDA(cudaFree(p));
    });
}
int rs_memset_async(rs_ctx *ctx, void *p, int32_t value, int64_t bytes) {
    return guard([&] {
        need(ctx, "rs_memset_async");
        if (bytes > 0) RS_CUDA(cudaMemsetAsync(p, value, (size_t)bytes, ctx->stream));
    });
}
int rs_memcpy_h2d(rs_ctx *ctx, void *dst_dev, const void *src, int64_t bytes) {
    return guard([&] {
        need(ctx, "rs_memcpy_h2d");
        if (bytes > 0) RS_CUDA(cudaMemcpyAsync(dst_dev, src, (size_t)bytes, cudaMemcpyHostToDevice, ctx->stream));
        RS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int rs_memcpy_d2h(rs_ctx *ctx, void *dst, const void *src_dev, int64_t bytes) {
    return guard([&] {
        need(ctx, "rs_memcpy_d2h");
        if (bytes > 0) RS_CUDA(cudaMemcpyAsync(dst, src_dev, (size_t)bytes, cudaMemcpyDeviceToHost, ctx->stream));
        RS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
