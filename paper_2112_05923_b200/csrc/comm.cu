// comm.cu -- the tournament's only cross-GPU traffic:
// score all-gather + identical ranking on every rank, and the elite-weight
// broadcast, both as NCCL collectives over NVLink on the context's stream.
// NCCL is resolved at run time (dlopen libnccl.so.2) so single-GPU users of
// the library carry no NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "prb_internal.h"

using namespace prb;

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
    n.AllGather = (decltype(n.AllGather))dlsym(n.h, "ncclAllGather");
    n.Broadcast = (decltype(n.Broadcast))dlsym(n.h, "ncclBroadcast");
    n.GroupStart = (decltype(n.GroupStart))dlsym(n.h, "ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.h, "ncclGroupEnd");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
  });
  PRB_REQUIRE(n.h && n.GetUniqueId && n.CommInitRank && n.AllGather && n.Broadcast, PRB_ERR_CUDA,
              "NCCL (libnccl.so.2) is not available");
  return n;
}

#define PRB_NCCL(call)                                                                         \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      fail(PRB_ERR_CUDA, std::string(#call) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r_) : "nccl")); \
  } while (0)

}  // namespace

struct prb_comm_s {
  prb_ctx_s* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

extern "C" {

int prb_comm_unique_id(uint8_t id[128]) {
  return guard([&] {
    ncclUniqueId u;
    PRB_NCCL(nccl().GetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
  });
}

int prb_comm_init(prb_ctx ctx, const uint8_t id[128], int nranks, int rank, prb_comm* out) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && id && out, PRB_ERR_USAGE, "prb_comm_init: NULL argument");
    PRB_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, PRB_ERR_CONFIG, "prb_comm_init: bad rank/nranks");
    PRB_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    auto* c = new prb_comm_s;
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    PRB_NCCL(nccl().CommInitRank(&c->comm, nranks, u, rank));
    *out = c;
  });
}

int prb_comm_destroy(prb_comm c) {
  return guard([&] {
    DeviceScope dev_(c ? c->ctx : nullptr);
    if (!c) return;
    if (c->comm) nccl().CommDestroy(c->comm);
    delete c;
  });
}

int prb_leaderboard_rank(prb_ctx ctx, const double* d_scores, const uint64_t* d_seqs, size_t n, size_t capacity,
                         int32_t* d_order, int32_t* d_count);

int prb_leaderboard_allgather_rank(prb_comm c, const double* d_scores, const uint64_t* d_seqs, const int64_t* d_ids,
                                   size_t n_local, size_t capacity, double* d_all_scores, uint64_t* d_all_seqs,
                                   int64_t* d_all_ids, int32_t* d_order, int32_t* d_count) {
  return guard([&] {
    DeviceScope dev_(c ? c->ctx : nullptr);
    PRB_REQUIRE(c && d_scores && d_seqs && d_ids && d_all_scores && d_all_seqs && d_all_ids && d_order && d_count,
                PRB_ERR_USAGE, "prb_leaderboard_allgather_rank: NULL argument");
    cudaStream_t s = c->ctx->stream;
    Nccl& n = nccl();
    PRB_NCCL(n.GroupStart());
    PRB_NCCL(n.AllGather(d_scores, d_all_scores, n_local, ncclFloat64, c->comm, s));
    PRB_NCCL(n.AllGather(d_seqs, d_all_seqs, n_local, ncclUint64, c->comm, s));
    PRB_NCCL(n.AllGather(d_ids, d_all_ids, n_local, ncclInt64, c->comm, s));
    PRB_NCCL(n.GroupEnd());
    const int rc = prb_leaderboard_rank(c->ctx, d_all_scores, d_all_seqs, n_local * (size_t)c->nranks, capacity,
                                        d_order, d_count);
    if (rc) fail(rc, prb_last_error());
  });
}

int prb_agent_broadcast(prb_comm c, prb_agent a, int root) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(c && a, PRB_ERR_USAGE, "prb_agent_broadcast: NULL argument");
    PRB_REQUIRE(root >= 0 && root < c->nranks, PRB_ERR_CONFIG, "prb_agent_broadcast: bad root");
    cudaStream_t s = c->ctx->stream;
    if (a->ctx->stream != s) a->ctx->sync();
    Nccl& n = nccl();
    PRB_NCCL(n.GroupStart());
    PRB_NCCL(n.Broadcast(a->d_params.p, a->d_params.p, a->P, ncclFloat32, root, c->comm, s));
    PRB_NCCL(n.Broadcast(a->d_m.p, a->d_m.p, a->P, ncclFloat32, root, c->comm, s));
    PRB_NCCL(n.Broadcast(a->d_v.p, a->d_v.p, a->P, ncclFloat32, root, c->comm, s));
    PRB_NCCL(n.Broadcast(a->d_t.p, a->d_t.p, 1, ncclInt64, root, c->comm, s));
    PRB_NCCL(n.GroupEnd());
    c->ctx->sync();
  });
}

}  // extern "C"
