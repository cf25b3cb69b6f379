// wr_ctx.cu - a9 the library-owned multi-GPU context (SURVEY §8(b)
// wr_ctx_create / wr_ctx_free, §8(e)): one context per process and GPU,
// owning an NCCL communicator over the world of ranks. The exchange steps
// of the sharded path run inside libwr on the caller's stream:
//   * wr_route_orders with opts.ctx: sources and orders sharded over the
//     world (wr_orders_plan / _local / _finish), ONE ncclAllGather of the
//     owned D entries between the relaxation and the routing phases, then
//     the ranks' result blocks exchanged (grouped ncclBroadcast, no padding)
//     so every rank holds all B results;
//   * wr_bf_batch with opts.ctx and opts.shard = 1: each rank relaxes its
//     contiguous block of the sources and the dist / pred row blocks are
//     exchanged the same way (§4.7: the V x N batch of sources
//     processed simultaneously, here split over GPUs).
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy torch has
// already loaded, or the system one), so libwr has no link-time dependency
// and a process that never creates a context never touches NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "wr_internal.cuh"

struct wr_ctx {
    int rank = 0, world = 1, device = 0;
    ncclComm_t comm = nullptr;
};

namespace wr {

namespace {
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char *name) { return dlsym(h, name); };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
        api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.Broadcast &&
                 api.GroupStart && api.GroupEnd && api.GetErrorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess)
        WR_THROW(WR_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

NcclApi &nccl_or_throw() {
    NcclApi &a = nccl();
    if (!a.ok) WR_THROW(WR_ENCCL, "NCCL unavailable: " + a.why);
    return a;
}
}  // namespace

int ctx_rank(const wr_ctx *c) { return c ? c->rank : 0; }
int ctx_world(const wr_ctx *c) { return c ? c->world : 1; }

void ctx_allgather(const wr_ctx *c, const void *send, void *recv, size_t bytes, cudaStream_t st) {
    NcclApi &a = nccl_or_throw();
    nccl_check(a.AllGather(send, recv, bytes, ncclUint8, c->comm, st), "ncclAllGather");
}

// Every rank r owns bytes [off[r], off[r+1]) of buf (same layout on all
// ranks); afterwards every rank holds the whole buffer. Grouped broadcasts
// move each block from its owner in place: no padding to the largest block.
void ctx_share_blocks(const wr_ctx *c, void *buf, const int64_t *off, cudaStream_t st) {
    NcclApi &a = nccl_or_throw();
    nccl_check(a.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < c->world; ++r) {
        const size_t n = (size_t)(off[r + 1] - off[r]);
        if (n == 0) continue;
        char *p = (char *)buf + off[r];
        nccl_check(a.Broadcast(p, p, n, ncclUint8, r, c->comm, st), "ncclBroadcast");
    }
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

}  // namespace wr

extern "C" {

wr_status wr_nccl_unique_id(void *uid_out) {
    return wr::guarded([&]() -> wr_status {
        if (!uid_out) return wr::fail(WR_EINVAL, "wr_nccl_unique_id: null output");
        ncclUniqueId id;
        wr::nccl_check(wr::nccl_or_throw().GetUniqueId(&id), "ncclGetUniqueId");
        static_assert(sizeof(ncclUniqueId) == WR_NCCL_UID_BYTES, "unique id size");
        memcpy(uid_out, &id, sizeof(id));
        return WR_OK;
    });
}

wr_status wr_ctx_create(int32_t rank, int32_t world, const void *nccl_uid, int32_t device, wr_ctx **out) {
    return wr::guarded([&]() -> wr_status {
        if (!out || world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_uid))
            return wr::fail(WR_EINVAL, "wr_ctx_create: bad arguments");
        int ndev = 0;
        WR_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) return wr::fail(WR_EINVAL, "wr_ctx_create: device");
        WR_CUDA(cudaSetDevice(device));
        auto &a = wr::nccl_or_throw();
        ncclUniqueId id;
        if (nccl_uid) memcpy(&id, nccl_uid, sizeof(id));
        else wr::nccl_check(a.GetUniqueId(&id), "ncclGetUniqueId");   // world 1: a private communicator
        auto c = new wr_ctx;
        c->rank = rank;
        c->world = world;
        c->device = device;
        ncclResult_t r = a.CommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            delete c;
            return wr::fail(WR_ENCCL, std::string("ncclCommInitRank: ") + a.GetErrorString(r));
        }
        *out = c;
        return WR_OK;
    });
}

wr_status wr_ctx_free(wr_ctx *c) {
    if (!c) return WR_OK;
    return wr::guarded([&]() -> wr_status {
        WR_CUDA(cudaSetDevice(c->device));
        if (c->comm) wr::nccl_check(wr::nccl_or_throw().CommDestroy(c->comm), "ncclCommDestroy");
        delete c;
        return WR_OK;
    });
}

wr_status wr_ctx_info(const wr_ctx *c, int32_t *rank, int32_t *world, int32_t *device) {
    if (!c) return wr::fail(WR_EINVAL, "wr_ctx_info: null context");
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    if (device) *device = c->device;
    return WR_OK;
}

}  // extern "C"
