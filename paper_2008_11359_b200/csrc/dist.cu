// dist.cu -- multi-GPU plumbing for destination-row sharding (SURVEY §8(a) row
// a6, §8(e)).  The paper is single-GPU and lists multi-GPU as future
// work; the exchange step here is the only collective the sharded
// path needs: every rank owns dst rows [lo, hi) and the matching rows of X, and
// gathers the source features of all ranks (all-gather-v of row blocks) over
// NVLink / NVSwitch before running its local fg_spmm / fg_sddmm.  Edge softmax
// and u_mul_e need no communication: all in-edges of a destination live on its
// owner.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") so the library has
// no link-time NCCL dependency and shares the copy torch already loaded.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "fg_internal.h"

struct fg_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0;
};

namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    bool ok = false;
};

NcclApi& api() {
    static NcclApi a;
    static bool tried = false;
    if (tried) return a;
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
        a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
        if (a.h) break;
    }
    if (!a.h) return a;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(a.h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(a.h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(dlsym(a.h, "ncclBroadcast"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(a.h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(a.h, "ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(a.h, "ncclGetErrorString"));
    a.CommCount = reinterpret_cast<decltype(a.CommCount)>(dlsym(a.h, "ncclCommCount"));
    a.CommUserRank = reinterpret_cast<decltype(a.CommUserRank)>(dlsym(a.h, "ncclCommUserRank"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Broadcast && a.GroupStart && a.GroupEnd &&
           a.GetErrorString;
    return a;
}

fg_status nccl_fail(const char* what, ncclResult_t r) {
    return fgk::set_error(FG_ENCCL, "%s: %s", what, api().GetErrorString ? api().GetErrorString(r) : "?");
}
}  // namespace

extern "C" fg_status fg_comm_unique_id(void* uid) {
    if (!uid) return fgk::set_error(FG_EINVAL, "fg_comm_unique_id: NULL");
    NcclApi& a = api();
    if (!a.ok) return fgk::set_error(FG_ENCCL, "fg_comm_unique_id: libnccl.so.2 not loadable");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    ncclUniqueId id;
    ncclResult_t r = a.GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
    std::memcpy(uid, &id, 128);
    return FG_OK;
}

extern "C" fg_status fg_comm_init(const void* uid, int nranks, int rank, fg_comm** out) {
    if (!uid || !out) return fgk::set_error(FG_EINVAL, "fg_comm_init: NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fgk::set_error(FG_EINVAL, "fg_comm_init: bad rank/nranks");
    NcclApi& a = api();
    if (!a.ok) return fgk::set_error(FG_ENCCL, "fg_comm_init: libnccl.so.2 not loadable");
    ncclUniqueId id;
    std::memcpy(&id, uid, 128);
    fg_comm* c = new fg_comm();
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = a.CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail("ncclCommInitRank", r);
    }
    *out = c;
    return FG_OK;
}

extern "C" fg_status fg_comm_info(const fg_comm* c, int* nranks, int* rank) {
    if (!c || !nranks || !rank) return fgk::set_error(FG_EINVAL, "fg_comm_info: NULL argument");
    NcclApi& a = api();
    if (!a.CommCount || !a.CommUserRank) return fgk::set_error(FG_ENCCL, "fg_comm_info: ncclCommCount unavailable");
    ncclResult_t r = a.CommCount(c->comm, nranks);
    if (r == ncclSuccess) r = a.CommUserRank(c->comm, rank);
    if (r != ncclSuccess) return nccl_fail("ncclCommCount/UserRank", r);
    return FG_OK;
}

extern "C" fg_status fg_comm_destroy(fg_comm* c) {
    if (!c) return fgk::set_error(FG_EINVAL, "fg_comm_destroy: NULL");
    if (c->comm) api().CommDestroy(c->comm);
    delete c;
    return FG_OK;
}

extern "C" fg_status fg_allgather_rows(fg_comm* c, const int64_t* off, int64_t row_elems, const float* X_local,
                                       float* X_full, fg_stream stream) {
    if (!c || !off || !X_full) return fgk::set_error(FG_EINVAL, "fg_allgather_rows: NULL argument");
    if (row_elems < 0) return fgk::set_error(FG_ESHAPE, "fg_allgather_rows: row_elems < 0");
    for (int r = 0; r < c->nranks; ++r)
        if (off[r + 1] < off[r]) return fgk::set_error(FG_ESHAPE, "fg_allgather_rows: offsets decrease");
    NcclApi& a = api();
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    ncclResult_t r = a.GroupStart();
    if (r != ncclSuccess) return nccl_fail("ncclGroupStart", r);
    for (int root = 0; root < c->nranks; ++root) {
        const size_t count = size_t(off[root + 1] - off[root]) * size_t(row_elems);
        float* dst = X_full + off[root] * row_elems;
        const void* src = (root == c->rank) ? static_cast<const void*>(X_local ? X_local : dst) : dst;
        r = a.Broadcast(src, dst, count, ncclFloat32, root, c->comm, st);
        if (r != ncclSuccess) {
            a.GroupEnd();
            return nccl_fail("ncclBroadcast", r);
        }
    }
    r = a.GroupEnd();
    if (r != ncclSuccess) return nccl_fail("ncclGroupEnd", r);
    return FG_OK;
}

// ---------------------------------------------------------------- sharded ops
// The dst-row-sharded forms of gSpMM / gSDDMM: the one
// exchange step (all-gather of the source-feature row blocks over NVLink) then
// the unchanged local kernel on this rank's rows, both enqueued on `stream`.
extern "C" fg_status fg_dist_spmm(const fg_graph* local, fg_comm* c, const int64_t* shard_offsets, fg_msg_op msg,
                                  fg_reduce_op red, int H, int D, const float* X_local, float* X_full, const float* E,
                                  const float* W, int d_in, const float* X_dst, float* out_local, int32_t* arg_u,
                                  int32_t* arg_e, void* workspace, size_t workspace_bytes, fg_stream stream) {
    if (!local || !c || !shard_offsets || !X_full) return fgk::set_error(FG_EINVAL, "fg_dist_spmm: NULL argument");
    if (msg == FG_MSG_COPY_E) return fgk::set_error(FG_EUNSUPPORTED, "fg_dist_spmm: copy_e gathers no source rows");
    const int64_t row_elems = (msg == FG_MSG_MLP) ? int64_t(d_in) : int64_t(H) * D;
    // every argument check of the local op runs BEFORE the collective is enqueued:
    // a non-OK status means nothing was launched and X_full is untouched
    fg_status s = fgk::check_spmm(local, msg, red, H, D, X_full, E, W, d_in, X_dst, out_local, arg_u, arg_e);
    if (s != FG_OK) return s;
    s = fg_allgather_rows(c, shard_offsets, row_elems, X_local, X_full, stream);
    if (s != FG_OK) return s;
    return fg_spmm(local, msg, red, H, D, X_full, E, W, d_in, X_dst, out_local, arg_u, arg_e, workspace,
                   workspace_bytes, stream);
}

extern "C" fg_status fg_dist_sddmm(const fg_graph* local, fg_comm* c, const int64_t* shard_offsets, fg_edge_op op,
                                   int H, int D, const float* X_local, float* X_full, const float* Y_local,
                                   float* out_local, fg_stream stream) {
    if (!local || !c || !shard_offsets || !X_full) return fgk::set_error(FG_EINVAL, "fg_dist_sddmm: NULL argument");
    fg_status s = fgk::check_sddmm(local, op, H, D, X_full, Y_local, out_local);
    if (s != FG_OK) return s;
    s = fg_allgather_rows(c, shard_offsets, int64_t(H) * D, X_local, X_full, stream);
    if (s != FG_OK) return s;
    return fg_sddmm(local, op, H, D, X_full, Y_local, out_local, stream);
}
