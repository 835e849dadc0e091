// comm.cpp — multi-GPU exchange for token-sharded runs.
//
// The only exchange step of the method: the column max m_d = MAX over ranks of
// each rank's local max (a7), as an in-place all-reduce MAX over D uint32
// abs-bit patterns (bit-exact, order-independent), plus the metric sums/maxima.
// NCCL is loaded with dlopen at first use (torch has usually loaded the wheel's
// libnccl.so.2 already; KVQ_NCCL_LIB overrides the path), so libkvq.so itself
// has no link-time NCCL dependency and single-GPU use never touches it.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include <nccl.h>

#include "kvq_internal.h"

struct kvq_comm_s {
    ncclComm_t comm;   // nullptr for a peer-backed communicator
    int nranks;
    int rank;
    kvq_peer_t peer;   // kvq_comm_from_peer: every collective goes through peer memory (peer.cu), no NCCL
};

namespace kvq {
namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
};

NcclApi &api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *env = std::getenv("KVQ_NCCL_LIB");
        const char *names[] = {env, "libnccl.so.2", "libnccl.so"};
        void *h = nullptr;
        for (const char *n : names) {
            if (!n) continue;
            h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            a.err = std::string("cannot dlopen NCCL (set KVQ_NCCL_LIB): ") + dlerror();
            return;
        }
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
        a.getErrorString = (decltype(a.getErrorString))dlsym(h, "ncclGetErrorString");
        a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
        a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.getErrorString &&
               a.groupStart && a.groupEnd;
        if (!a.ok) a.err = "NCCL library lacks required symbols";
    });
    return a;
}

kvq_status nccl_fail(ncclResult_t r, const char *what) {
    NcclApi &a = api();
    return fail(KVQ_ERR_NCCL, std::string(what) + ": " + (a.getErrorString ? a.getErrorString(r) : "?"));
}

kvq_status allreduce(kvq_comm_t comm, void *buf, size_t count, ncclDataType_t ty, ncclRedOp_t op, cudaStream_t s,
                     const char *what) {
    NcclApi &a = api();
    if (!a.ok) return fail(KVQ_ERR_NCCL, a.err);
    ncclResult_t r = a.allReduce(buf, buf, count, ty, op, comm->comm, s);
    if (r != ncclSuccess) return nccl_fail(r, what);
    return KVQ_OK;
}

}  // namespace

kvq_peer_t comm_peer(kvq_comm_t comm) { return comm ? comm->peer : nullptr; }

kvq_status comm_allreduce_max_u32(kvq_comm_t comm, uint32_t *buf, size_t count, cudaStream_t s) {
    if (comm->peer) return peer_allreduce_max_u32(comm->peer, buf, count, s);
    return allreduce(comm, buf, count, ncclUint32, ncclMax, s, "allreduce(max,u32)");
}
kvq_status comm_allreduce_sum_f64(kvq_comm_t comm, double *buf, size_t count, cudaStream_t s) {
    return allreduce(comm, buf, count, ncclFloat64, ncclSum, s, "allreduce(sum,f64)");
}
kvq_status comm_allreduce_max_u64(kvq_comm_t comm, uint64_t *buf, size_t count, cudaStream_t s) {
    return allreduce(comm, buf, count, ncclUint64, ncclMax, s, "allreduce(max,u64)");
}
// The metric partials (a5/a6): fp64 sums (SUM) and u64 bit-pattern maxima (MAX)
// in ONE NCCL group, i.e. one fused launch instead of two per step.
kvq_status comm_allreduce_metrics(kvq_comm_t comm, double *sums, size_t nsum, uint64_t *maxes, size_t nmax,
                                  cudaStream_t s) {
    if (comm->peer) return peer_allreduce_metrics(comm->peer, sums, nsum, maxes, nmax, s);
    NcclApi &a = api();
    if (!a.ok) return fail(KVQ_ERR_NCCL, a.err);
    ncclResult_t r = a.groupStart();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    kvq_status st = allreduce(comm, sums, nsum, ncclFloat64, ncclSum, s, "allreduce(sum,f64)");
    if (st == KVQ_OK) st = allreduce(comm, maxes, nmax, ncclUint64, ncclMax, s, "allreduce(max,u64)");
    r = a.groupEnd();
    if (st != KVQ_OK) return st;
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
    return KVQ_OK;
}

}  // namespace kvq

extern "C" kvq_status kvq_comm_unique_id(void *out_id128) {
    KVQ_NVTX("kvq_comm_unique_id");
    using namespace kvq;
    if (!out_id128) return fail(KVQ_ERR_INVALID_VALUE, "kvq_comm_unique_id: NULL");
    NcclApi &a = api();
    if (!a.ok) return fail(KVQ_ERR_NCCL, a.err);
    ncclUniqueId id;
    ncclResult_t r = a.getUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(out_id128, &id, sizeof(id));
    return KVQ_OK;
}

extern "C" kvq_status kvq_comm_init(kvq_comm_t *out, const void *id128, int nranks, int rank) {
    KVQ_NVTX("kvq_comm_init");
    using namespace kvq;
    if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(KVQ_ERR_INVALID_VALUE, "kvq_comm_init: invalid argument");
    *out = nullptr;
    if (kvq_status st = device_ok(); st != KVQ_OK) return st;
    NcclApi &a = api();
    if (!a.ok) return fail(KVQ_ERR_NCCL, a.err);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    kvq_comm_s *c = new kvq_comm_s{nullptr, nranks, rank, nullptr};
    ncclResult_t r = a.commInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *out = c;
    return KVQ_OK;
}

extern "C" kvq_status kvq_comm_from_peer(kvq_comm_t *out, kvq_peer_t p) {
    KVQ_NVTX("kvq_comm_from_peer");
    using namespace kvq;
    if (!out || !p) return fail(KVQ_ERR_INVALID_VALUE, "kvq_comm_from_peer: NULL");
    if (!peer_ready(p)) return fail(KVQ_ERR_INVALID_VALUE, "kvq_comm_from_peer: call kvq_peer_open first");
    *out = new kvq_comm_s{nullptr, peer_nranks(p), peer_rank(p), p};
    return KVQ_OK;
}

extern "C" kvq_status kvq_comm_destroy(kvq_comm_t comm) {
    KVQ_NVTX("kvq_comm_destroy");
    using namespace kvq;
    if (!comm) return KVQ_OK;
    if (comm->peer) {  // the peer itself belongs to the caller (kvq_peer_destroy)
        delete comm;
        return KVQ_OK;
    }
    NcclApi &a = api();
    kvq_status st = KVQ_OK;
    if (a.ok) {
        ncclResult_t r = a.commDestroy(comm->comm);
        if (r != ncclSuccess) st = nccl_fail(r, "ncclCommDestroy");
    }
    delete comm;
    return st;
}
