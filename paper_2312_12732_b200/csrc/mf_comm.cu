// mf_comm.cu -- the exchange layer of the product-sharded path (SURVEY.md §8e,
// row a6; the paper's "each product can be done recursively", PAPER.md L203,
// makes the R^L leaf products independent, and the post-addition is linear, so
// partial C sums over disjoint product sets add up to C).
//
// mf_dgemm talks to a Comm, never to NCCL directly.  Two transports:
//  * NcclComm -- one process per GPU, NCCL over NVLink 5 / NVSwitch (the
//    product path; libnccl.so.2 is dlopen'ed, torch's copy when loaded);
//  * LoopComm -- N ranks as N host threads of ONE process (same device or
//    peer-accessible devices).  Every collective is a host rendezvous of the N
//    threads followed by stream-ordered copies / a summation kernel that the
//    receiving rank enqueues on its own stream after cudaStreamWaitEvent on the
//    senders' "ready" events.  No kernel ever waits on another rank's kernel
//    (nothing spins on the GPU), so this is safe on one GPU; it exists so the
//    multi-rank schedule (who broadcasts, reduces, scatters what, in which
//    order, at which offsets) runs and is checked against the oracle where only
//    one GPU exists.  Sums are in ascending rank order (deterministic).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "mf_internal.h"

namespace mf {

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // Prefer the NCCL already loaded into the process (torch's), else the loader path.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.h = h;
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(h, "ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(h, "ncclCommDestroy");
    n.Reduce = (decltype(n.Reduce))dlsym(h, "ncclReduce");
    n.AllReduce = (decltype(n.AllReduce))dlsym(h, "ncclAllReduce");
    n.Broadcast = (decltype(n.Broadcast))dlsym(h, "ncclBroadcast");
    n.ReduceScatter = (decltype(n.ReduceScatter))dlsym(h, "ncclReduceScatter");
    n.AllGather = (decltype(n.AllGather))dlsym(h, "ncclAllGather");
    n.GroupStart = (decltype(n.GroupStart))dlsym(h, "ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))dlsym(h, "ncclGroupEnd");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(h, "ncclGetErrorString");
  });
  return n.h && n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Reduce && n.AllReduce &&
                 n.Broadcast && n.ReduceScatter && n.AllGather && n.GroupStart && n.GroupEnd
             ? &n
             : nullptr;
}

static mf_status nccl_fail(Nccl* n, ncclResult_t r, const char* what) {
  return fail(MF_ERR_NCCL, "%s: %s", what, n && n->GetErrorString ? n->GetErrorString(r) : "?");
}

#define MF_NCCL(call, what)                                   \
  do {                                                        \
    ncclResult_t r_ = (call);                                 \
    if (r_ != ncclSuccess) return nccl_fail(nc_, r_, what);   \
  } while (0)

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  Nccl* nc_ = nullptr;
  const char* kind() const override { return "nccl"; }
  mf_status bcast(void* buf, size_t count, int root, cudaStream_t s) override {
    MF_NCCL(nc_->Broadcast(buf, buf, count, ncclDouble, root, c, s), "ncclBroadcast");
    return MF_OK;
  }
  mf_status reduce(const double* send, double* recv, size_t count, int root,
                   cudaStream_t s) override {
    MF_NCCL(nc_->Reduce(send, recv, count, ncclDouble, ncclSum, root, c, s), "ncclReduce");
    return MF_OK;
  }
  mf_status allreduce(const double* send, double* recv, size_t count, cudaStream_t s) override {
    MF_NCCL(nc_->AllReduce(send, recv, count, ncclDouble, ncclSum, c, s), "ncclAllReduce");
    return MF_OK;
  }
  mf_status reduce_scatter(const double* send, double* recv, size_t recvcount,
                           cudaStream_t s) override {
    MF_NCCL(nc_->ReduceScatter(send, recv, recvcount, ncclDouble, ncclSum, c, s),
            "ncclReduceScatter");
    return MF_OK;
  }
  mf_status allgather(const double* send, double* recv, size_t sendcount,
                      cudaStream_t s) override {
    MF_NCCL(nc_->AllGather(send, recv, sendcount, ncclDouble, c, s), "ncclAllGather");
    return MF_OK;
  }
  mf_status group_start() override {
    MF_NCCL(nc_->GroupStart(), "ncclGroupStart");
    return MF_OK;
  }
  mf_status group_end() override {
    MF_NCCL(nc_->GroupEnd(), "ncclGroupEnd");
    return MF_OK;
  }
  ~NcclComm() override {
    if (c && nc_) nc_->CommDestroy(c);
  }
};

// ------------------------------------------------------ in-process loopback ranks
constexpr int kLoopMaxRanks = 16;

struct SumArgs {
  const double* in[kLoopMaxRanks];
  int n;
};

// out[i] = in[0][i] + in[1][i] + ... (ascending rank; out may alias an input)
__global__ void __launch_bounds__(256) loop_sum_kernel(double* out, SumArgs a, size_t count) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    double acc = a.in[0][i];
    for (int k = 1; k < a.n; ++k) acc += a.in[k][i];
    out[i] = acc;
  }
}

struct LoopGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  int refs = 0;
  struct Slot {
    const void* send = nullptr;
    void* recv = nullptr;
  };
  std::vector<Slot> slot;
  std::vector<cudaEvent_t> ready, done;  // per rank, created by the rank's thread

  // all n ranks arrive (or the group breaks after a timeout: a rank failed
  // before reaching this collective)
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct LoopComm final : Comm {
  LoopGroup* g = nullptr;
  const char* kind() const override { return "loopback"; }

  mf_status ensure_events() {
    if (g->ready[rank]) return MF_OK;
    if (cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming) != cudaSuccess)
      return fail(MF_ERR_CUDA, "loopback communicator: cudaEventCreate");
    return MF_OK;
  }

  // One collective: publish (send, recv) and a "ready" event after this rank's
  // prior work on s; rendezvous; wait for every peer's ready event; enqueue
  // this rank's part (body); record "done"; rendezvous; wait for every peer's
  // done event, so no rank reuses a buffer a peer is still reading.
  template <class Body>
  mf_status run(const void* send, void* recv, cudaStream_t s, const char* what, Body&& body) {
    mf_status st = ensure_events();
    if (st != MF_OK) return st;
    // publish: every peer finished reading the slots of the previous
    // collective before its second rendezvous
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->slot[rank].send = send;
      g->slot[rank].recv = recv;
    }
    if (cudaEventRecord(g->ready[rank], s) != cudaSuccess)
      return fail(MF_ERR_CUDA, "loopback %s: cudaEventRecord", what);
    if (!g->barrier()) return fail(MF_ERR_NCCL, "loopback %s: a peer rank did not arrive", what);
    for (int k = 0; k < size; ++k)
      if (k != rank && cudaStreamWaitEvent(s, g->ready[k], 0) != cudaSuccess)
        return fail(MF_ERR_CUDA, "loopback %s: cudaStreamWaitEvent", what);
    const cudaError_t e = body();
    if (e != cudaSuccess) {
      g->barrier();  // let the peers finish this collective
      return fail(MF_ERR_CUDA, "loopback %s: %s", what, cudaGetErrorString(e));
    }
    if (cudaEventRecord(g->done[rank], s) != cudaSuccess)
      return fail(MF_ERR_CUDA, "loopback %s: cudaEventRecord", what);
    if (!g->barrier()) return fail(MF_ERR_NCCL, "loopback %s: a peer rank did not arrive", what);
    // (re-recording is safe: a peer enqueues its waits on this rank's ready
    // event before the second rendezvous and on its done event before the
    // next collective's first, which this rank cannot pass before it)
    for (int k = 0; k < size; ++k)
      if (k != rank && cudaStreamWaitEvent(s, g->done[k], 0) != cudaSuccess)
        return fail(MF_ERR_CUDA, "loopback %s: cudaStreamWaitEvent", what);
    return MF_OK;
  }

  cudaError_t sum(double* out, size_t offset, size_t count, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    SumArgs a{};
    a.n = size;
    for (int k = 0; k < size; ++k) a.in[k] = static_cast<const double*>(g->slot[k].send) + offset;
    const int blocks = (int)std::min<size_t>((count + 255) / 256, 148 * 16);
    loop_sum_kernel<<<blocks, 256, 0, s>>>(out, a, count);
    return cudaGetLastError();
  }

  mf_status bcast(void* buf, size_t count, int root, cudaStream_t s) override {
    return run(buf, buf, s, "broadcast", [&]() -> cudaError_t {
      if (rank == root || count == 0) return cudaSuccess;
      return cudaMemcpyAsync(buf, g->slot[root].recv, count * sizeof(double), cudaMemcpyDefault, s);
    });
  }
  mf_status reduce(const double* send, double* recv, size_t count, int root,
                   cudaStream_t s) override {
    return run(send, recv, s, "reduce", [&]() -> cudaError_t {
      return rank == root ? sum(recv, 0, count, s) : cudaSuccess;
    });
  }
  mf_status allreduce(const double* send, double* recv, size_t count, cudaStream_t s) override {
    mf_status st = reduce(send, recv, count, 0, s);
    return st != MF_OK ? st : bcast(recv, count, 0, s);
  }
  mf_status reduce_scatter(const double* send, double* recv, size_t recvcount,
                           cudaStream_t s) override {
    return run(send, recv, s, "reduce-scatter", [&]() -> cudaError_t {
      return sum(recv, (size_t)rank * recvcount, recvcount, s);
    });
  }
  mf_status allgather(const double* send, double* recv, size_t sendcount,
                      cudaStream_t s) override {
    return run(send, recv, s, "all-gather", [&]() -> cudaError_t {
      for (int k = 0; k < size; ++k) {
        const double* src = static_cast<const double*>(g->slot[k].send);
        double* dst = recv + (size_t)k * sendcount;
        if (src == dst || sendcount == 0) continue;
        const cudaError_t e = cudaMemcpyAsync(dst, src, sendcount * sizeof(double), cudaMemcpyDefault, s);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    });
  }
  ~LoopComm() override {
    bool last = false;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      last = --g->refs == 0;
    }
    if (last) {
      for (cudaEvent_t e : g->ready)
        if (e) cudaEventDestroy(e);
      for (cudaEvent_t e : g->done)
        if (e) cudaEventDestroy(e);
      delete g;
    }
  }
};

Comm* comm_from(void* handle) {
  if (!handle) return nullptr;
  Comm* c = static_cast<Comm*>(handle);
  return c->magic == kCommMagic ? c : nullptr;
}

}  // namespace mf

using namespace mf;

extern "C" {

mf_status mf_nccl_unique_id(void* id_out) {
  Nccl* nc = nccl();
  if (!nc) return fail(MF_ERR_NCCL, "libnccl.so.2 could not be loaded");
  if (!id_out) return fail(MF_ERR_INVALID_ARG, "id_out is NULL");
  ncclUniqueId id;
  ncclResult_t r = nc->GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(nc, r, "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof id);
  return MF_OK;
}

mf_status mf_nccl_comm_create(void** comm_out, const void* id, int32_t rank, int32_t nranks) {
  Nccl* nc = nccl();
  if (!nc) return fail(MF_ERR_NCCL, "libnccl.so.2 could not be loaded");
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(MF_ERR_INVALID_ARG, "bad argument");
  *comm_out = nullptr;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  NcclComm* c = new (std::nothrow) NcclComm();
  if (!c) return fail(MF_ERR_OUT_OF_MEMORY, "host allocation");
  c->nc_ = nc;
  c->rank = rank;
  c->size = nranks;
  ncclResult_t r = nc->CommInitRank(&c->c, nranks, uid, rank);
  if (r != ncclSuccess) {
    c->c = nullptr;
    delete c;
    return nccl_fail(nc, r, "ncclCommInitRank");
  }
  *comm_out = static_cast<Comm*>(c);
  return MF_OK;
}

mf_status mf_loop_comm_create(int32_t nranks, void** comms_out) {
  if (!comms_out || nranks < 1 || nranks > kLoopMaxRanks)
    return fail(MF_ERR_INVALID_ARG, "nranks must be in [1, %d] and comms_out non-NULL", kLoopMaxRanks);
  LoopGroup* g = new (std::nothrow) LoopGroup();
  if (!g) return fail(MF_ERR_OUT_OF_MEMORY, "host allocation");
  g->n = nranks;
  g->slot.resize(nranks);
  g->ready.assign(nranks, nullptr);
  g->done.assign(nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    LoopComm* c = new (std::nothrow) LoopComm();
    if (!c) {
      for (int k = 0; k < r; ++k) delete static_cast<Comm*>(comms_out[k]);
      if (r == 0) delete g;
      return fail(MF_ERR_OUT_OF_MEMORY, "host allocation");
    }
    c->g = g;
    c->rank = r;
    c->size = nranks;
    ++g->refs;
    comms_out[r] = static_cast<Comm*>(c);
  }
  return MF_OK;
}

mf_status mf_comm_info(void* comm, int32_t* rank, int32_t* nranks, int32_t* kind) {
  Comm* c = comm_from(comm);
  if (!c) return fail(MF_ERR_INVALID_ARG, "not a communicator handle of this library");
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->size;
  if (kind) *kind = strcmp(c->kind(), "nccl") == 0 ? MF_COMM_NCCL : MF_COMM_LOOPBACK;
  return MF_OK;
}

mf_status mf_comm_destroy(void* comm) {
  if (!comm) return MF_OK;
  Comm* c = comm_from(comm);
  if (!c) return fail(MF_ERR_INVALID_ARG, "not a communicator handle of this library");
  c->magic = 0;
  delete c;
  return MF_OK;
}

mf_status mf_nccl_comm_destroy(void* comm) { return mf_comm_destroy(comm); }

}  // extern "C"
