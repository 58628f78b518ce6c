// comm.cu -- NCCL over NVLink/NVSwitch for the multi-GPU path (PAPER.md P:572-574:
// "the partitioning of the tree among MPI processes ... the communication of needed data to
// perform the FMM interactions", one process per GPU).
//
// libnccl is resolved at run time (dlopen of libnccl.so.2, i.e. the copy PyTorch already loaded
// when present), so the library has no link-time NCCL dependency and single-GPU use never touches
// it.  Only the handful of collectives the path needs are wrapped.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>
#include <string>

#include "kernels.cuh"

namespace fmm {

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;  // optional
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  if (a.h) return a;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (a.h) break;
  }
  if (!a.h) throw Error(FMMBEM_E_NCCL, "cannot dlopen libnccl.so.2");
  auto sym = [&](const char* s) {
    void* p = dlsym(a.h, s);
    if (!p) throw Error(FMMBEM_E_NCCL, std::string("libnccl lacks ") + s);
    return p;
  };
  a.getUniqueId = (decltype(a.getUniqueId))sym("ncclGetUniqueId");
  a.commInitRank = (decltype(a.commInitRank))sym("ncclCommInitRank");
  a.commDestroy = (decltype(a.commDestroy))sym("ncclCommDestroy");
  a.commSplit = (decltype(a.commSplit))dlsym(a.h, "ncclCommSplit");
  a.allReduce = (decltype(a.allReduce))sym("ncclAllReduce");
  a.broadcast = (decltype(a.broadcast))sym("ncclBroadcast");
  a.allGather = (decltype(a.allGather))sym("ncclAllGather");
  a.send = (decltype(a.send))sym("ncclSend");
  a.recv = (decltype(a.recv))sym("ncclRecv");
  a.groupStart = (decltype(a.groupStart))sym("ncclGroupStart");
  a.groupEnd = (decltype(a.groupEnd))sym("ncclGroupEnd");
  a.errStr = (decltype(a.errStr))sym("ncclGetErrorString");
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(FMMBEM_E_NCCL, std::string(what) + ": " + api().errStr(r));
}

}  // namespace

void comm_unique_id(void* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  check(api().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(id128, &id, sizeof(id));
}

void comm_init(fmmbem_ctx* c, const void* id128) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t comm;
  check(api().commInitRank(&comm, c->opt.nranks, id, c->opt.rank), "ncclCommInitRank");
  c->comm = comm;
  if (api().commSplit) {  // collective over comm: every rank takes this branch (same libnccl)
    ncclComm_t c2 = nullptr;
    check(api().commSplit(comm, 0, c->opt.rank, &c2, nullptr), "ncclCommSplit");
    c->comm2 = c2;
  }
}

void comm_destroy(fmmbem_ctx* c) {
  if (c->comm2) api().commDestroy((ncclComm_t)c->comm2);
  if (c->comm) api().commDestroy((ncclComm_t)c->comm);
  c->comm = c->comm2 = nullptr;
}

void comm_allreduce_f32(fmmbem_ctx* c, float* buf, size_t n, cudaStream_t s) {
  if (c->opt.nranks <= 1 || n == 0) return;
  check(api().allReduce(buf, buf, n, ncclFloat32, ncclSum, (ncclComm_t)c->comm, s), "ncclAllReduce");
}

void comm_allreduce_f64(fmmbem_ctx* c, double* buf, size_t n, cudaStream_t s) {
  if (c->opt.nranks <= 1 || n == 0) return;
  check(api().allReduce(buf, buf, n, ncclFloat64, ncclSum, (ncclComm_t)c->comm, s), "ncclAllReduce");
}

// full[offs[r] : offs[r+1]] <- rank r's slice, for every r (uneven slices: grouped broadcasts)
void comm_allgatherv_f32(fmmbem_ctx* c, const float* mine, float* full, const std::vector<int64_t>& offs,
                         cudaStream_t s, bool second) {
  const int R = c->opt.nranks;
  const ncclComm_t cm = (ncclComm_t)(second && c->comm2 ? c->comm2 : c->comm);
  check(api().groupStart(), "ncclGroupStart");
  for (int r = 0; r < R; ++r) {
    const size_t n = (size_t)(offs[r + 1] - offs[r]);
    if (!n) continue;
    check(api().broadcast(r == c->opt.rank ? (const void*)mine : (const void*)(full + offs[r]), full + offs[r], n,
                          ncclFloat32, r, cm, s),
          "ncclBroadcast");
  }
  check(api().groupEnd(), "ncclGroupEnd");
}

// grouped point-to-point exchange: sbuf[p] (scnt[p] floats) -> rank p, rbuf[p] <- rank p
void comm_sendrecv_f32(fmmbem_ctx* c, const std::vector<float*>& sbuf, const std::vector<size_t>& scnt,
                       const std::vector<float*>& rbuf, const std::vector<size_t>& rcnt, cudaStream_t s) {
  const int R = c->opt.nranks;
  check(api().groupStart(), "ncclGroupStart");
  for (int p = 0; p < R; ++p) {
    if (p == c->opt.rank) continue;
    if (scnt[p]) check(api().send(sbuf[p], scnt[p], ncclFloat32, p, (ncclComm_t)c->comm, s), "ncclSend");
    if (rcnt[p]) check(api().recv(rbuf[p], rcnt[p], ncclFloat32, p, (ncclComm_t)c->comm, s), "ncclRecv");
  }
  check(api().groupEnd(), "ncclGroupEnd");
}

// element-wise min / max of n doubles over ranks (device buffer, in place)
void comm_allreduce_f64_op(fmmbem_ctx* c, double* buf, size_t n, int op, cudaStream_t s) {
  if (c->opt.nranks <= 1 || n == 0) return;
  const ncclRedOp_t o = op < 0 ? ncclMin : (op > 0 ? ncclMax : ncclSum);
  check(api().allReduce(buf, buf, n, ncclFloat64, o, (ncclComm_t)c->comm, s), "ncclAllReduce");
}

// element-wise max of `n` uint32 values over the ranks (second: the caller-stream communicator)
void comm_allreduce_u32_max(fmmbem_ctx* c, unsigned* buf, size_t n, cudaStream_t s, bool second) {
  if (c->opt.nranks <= 1 || n == 0) return;
  const ncclComm_t cm = (ncclComm_t)(second && c->comm2 ? c->comm2 : c->comm);
  check(api().allReduce(buf, buf, n, ncclUint32, ncclMax, cm, s), "ncclAllReduce");
}

// every rank's `n` int64 values (device) -> all[r * n + k] (device)
void comm_allgather_i64(fmmbem_ctx* c, const int64_t* mine, int64_t* all, size_t n, cudaStream_t s) {
  check(api().allGather(mine, all, n, ncclInt64, (ncclComm_t)c->comm, s), "ncclAllGather");
}

// uneven all-gather of raw bytes: full[offs[r] : offs[r+1]] <- rank r's `mine` (grouped broadcasts)
void comm_allgatherv_bytes(fmmbem_ctx* c, const void* mine, void* full, const std::vector<size_t>& offs,
                           cudaStream_t s) {
  const int R = c->opt.nranks;
  char* f = static_cast<char*>(full);
  check(api().groupStart(), "ncclGroupStart");
  for (int r = 0; r < R; ++r) {
    const size_t n = offs[r + 1] - offs[r];
    if (!n) continue;
    check(api().broadcast(r == c->opt.rank ? mine : (const void*)(f + offs[r]), f + offs[r], n, ncclUint8, r,
                          (ncclComm_t)c->comm, s),
          "ncclBroadcast");
  }
  check(api().groupEnd(), "ncclGroupEnd");
}

// grouped point-to-point exchange of raw bytes (any peer may be this rank: local device copy)
void comm_alltoallv_bytes(fmmbem_ctx* c, const std::vector<const void*>& sbuf, const std::vector<size_t>& sbytes,
                          const std::vector<void*>& rbuf, const std::vector<size_t>& rbytes, cudaStream_t s,
                          bool second) {
  const int R = c->opt.nranks, me = c->opt.rank;
  const ncclComm_t cm = (ncclComm_t)(second && c->comm2 ? c->comm2 : c->comm);
  if (sbytes[me]) FMM_CUDA(cudaMemcpyAsync(rbuf[me], sbuf[me], sbytes[me], cudaMemcpyDeviceToDevice, s));
  if (R <= 1) return;
  check(api().groupStart(), "ncclGroupStart");
  for (int p = 0; p < R; ++p) {
    if (p == me) continue;
    if (sbytes[p]) check(api().send(sbuf[p], sbytes[p], ncclUint8, p, cm, s), "ncclSend");
    if (rbytes[p]) check(api().recv(rbuf[p], rbytes[p], ncclUint8, p, cm, s), "ncclRecv");
  }
  check(api().groupEnd(), "ncclGroupEnd");
}

// Contiguous split of n weighted items into `parts` ranges of (nearly) equal total weight:
// bounds[0] = 0, bounds[parts] = n, bounds[r] = first index whose prefix sum reaches r/parts of
// the total.  Pure host arithmetic, identical on every rank for identical inputs.
void split_costs(const double* cost, int64_t n, int parts, int64_t* bounds) {
  std::vector<double> pre(n + 1, 0.0);
  for (int64_t i = 0; i < n; ++i) pre[i + 1] = pre[i] + (cost[i] > 0 ? cost[i] : 0.0);
  const double tot = pre[n];
  bounds[0] = 0;
  int64_t k = 0;
  for (int r = 1; r < parts; ++r) {
    const double goal = tot * (double)r / (double)parts;
    while (k < n && pre[k + 1] <= goal) ++k;
    // choose the closer of k and k+1 as the cut
    int64_t cut = k;
    if (k < n && (goal - pre[k]) > (pre[k + 1] - goal)) cut = k + 1;
    bounds[r] = std::max<int64_t>(cut, bounds[r - 1]);
  }
  bounds[parts] = n;
}

}  // namespace fmm
