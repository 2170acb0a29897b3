// comm.cu — NCCL over NVLink for the multi-GPU path.
//
// libnccl.so.2 is resolved with dlopen at gc_comm_init time, so libgc loads
// (and runs single-GPU) without NCCL, and inside a PyTorch process it reuses
// the NCCL that torch already loaded (same soname).  Collectives run on the
// context stream:
//   triangle count  ncclAllReduce(uint64, sum, 1)
//   edge support    ncclAllReduce(uint32, sum, m)
//   k-truss peel    ncclAllGather of the removed-edge bitmap (per round; at a
//                   level start also the zero-support bitmap and an
//                   ncclAllReduce(min) of the smallest support left out);
//                   per chunk of a round's owned frontier, the decrements of
//                   other ranks' edges: counts by ncclAllGather, lists by
//                   grouped ncclBroadcast (allgatherv_i32)
#include <dlfcn.h>
#include <nccl.h>

#include "gc_internal.cuh"

namespace gcx {

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

NcclApi& api() {
    static NcclApi A;
    static bool tried = false;
    if (tried) return A;
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
        A.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (A.h) break;
    }
    if (!A.h) {
        A.why = std::string("dlopen(libnccl.so.2) failed: ") + (dlerror() ? dlerror() : "?");
        return A;
    }
#define SYM(field, name)                                                   \
    A.field = reinterpret_cast<decltype(A.field)>(dlsym(A.h, name));       \
    if (!A.field) {                                                        \
        A.why = std::string("NCCL symbol missing: ") + name;               \
        return A;                                                          \
    }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(CommAbort, "ncclCommAbort");
    SYM(AllReduce, "ncclAllReduce");
    SYM(AllGather, "ncclAllGather");
    SYM(Broadcast, "ncclBroadcast");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    A.ok = true;
    return A;
}

int nccl_fail(gc_ctx* c, ncclResult_t r, const char* what) {
    std::string msg = std::string("NCCL error in ") + what + ": " +
                      (api().GetErrorString ? api().GetErrorString(r) : "?");
    if (c) {
        c->poisoned = true;
        if (c->nccl && api().CommAbort) {
            api().CommAbort(static_cast<ncclComm_t>(c->nccl));
            c->nccl = nullptr;
        }
    }
    return fail(c, GC_ERR_NCCL, msg);
}

}  // namespace

int nccl_get_unique_id(void* id) {
    NcclApi& A = api();
    if (!A.ok) return GC_ERR_NCCL;
    ncclUniqueId uid;
    if (A.GetUniqueId(&uid) != ncclSuccess) return GC_ERR_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id, &uid, sizeof(uid));
    return GC_OK;
}

int nccl_init(gc_ctx* c, const void* id, int nranks, int rank) {
    NcclApi& A = api();
    if (!A.ok) return fail(c, GC_ERR_NCCL, A.why);
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    ncclResult_t r = A.CommInitRank(&comm, nranks, uid, rank);
    if (r != ncclSuccess) return nccl_fail(c, r, "ncclCommInitRank");
    c->nccl = comm;
    c->nranks = nranks;
    c->rank = rank;
    return GC_OK;
}

int nccl_destroy(gc_ctx* c) {
    if (c->nccl && api().ok) api().CommDestroy(static_cast<ncclComm_t>(c->nccl));
    c->nccl = nullptr;
    return GC_OK;
}

int allreduce_u64(gc_ctx* c, uint64_t* dev, size_t count) {
    ncclResult_t r = api().AllReduce(dev, dev, count, ncclUint64, ncclSum, static_cast<ncclComm_t>(c->nccl), c->stream);
    if (r != ncclSuccess) return nccl_fail(c, r, "ncclAllReduce(u64)");
    return GC_OK;
}

int allreduce_u32(gc_ctx* c, uint32_t* dev, size_t count) {
    ncclResult_t r = api().AllReduce(dev, dev, count, ncclUint32, ncclSum, static_cast<ncclComm_t>(c->nccl), c->stream);
    if (r != ncclSuccess) return nccl_fail(c, r, "ncclAllReduce(u32)");
    return GC_OK;
}

int allreduce_min_u32(gc_ctx* c, uint32_t* dev, size_t count) {
    ncclResult_t r = api().AllReduce(dev, dev, count, ncclUint32, ncclMin, static_cast<ncclComm_t>(c->nccl), c->stream);
    if (r != ncclSuccess) return nccl_fail(c, r, "ncclAllReduce(u32, min)");
    return GC_OK;
}

int allreduce_max_u32(gc_ctx* c, uint32_t* dev, size_t count) {
    ncclResult_t r = api().AllReduce(dev, dev, count, ncclUint32, ncclMax, static_cast<ncclComm_t>(c->nccl), c->stream);
    if (r != ncclSuccess) return nccl_fail(c, r, "ncclAllReduce(u32, max)");
    return GC_OK;
}

int allgather_u32(gc_ctx* c, const uint32_t* send, uint32_t* recv, size_t count_per_rank) {
    ncclResult_t r = api().AllGather(send, recv, count_per_rank, ncclUint32, static_cast<ncclComm_t>(c->nccl), c->stream);
    if (r != ncclSuccess) return nccl_fail(c, r, "ncclAllGather(u32)");
    return GC_OK;
}

// Variable-size allgather of int32 lists: rank r's counts[r] entries at
// send land at recv + offsets[r] on every rank (one ncclBroadcast per root,
// fused in a group).  counts / offsets are host arrays of nranks entries.
int allgatherv_i32(gc_ctx* c, const int32_t* send, int32_t* recv, const int64_t* counts, const int64_t* offsets) {
    NcclApi& A = api();
    ncclComm_t comm = static_cast<ncclComm_t>(c->nccl);
    ncclResult_t r = A.GroupStart();
    if (r != ncclSuccess) return nccl_fail(c, r, "ncclGroupStart");
    for (int root = 0; root < c->nranks; ++root) {
        if (counts[root] == 0) continue;
        r = A.Broadcast(root == c->rank ? send : recv + offsets[root], recv + offsets[root], (size_t)counts[root],
                        ncclInt32, root, comm, c->stream);
        if (r != ncclSuccess) {
            A.GroupEnd();
            return nccl_fail(c, r, "ncclBroadcast");
        }
    }
    r = A.GroupEnd();
    if (r != ncclSuccess) return nccl_fail(c, r, "ncclGroupEnd");
    return GC_OK;
}

}  // namespace gcx
