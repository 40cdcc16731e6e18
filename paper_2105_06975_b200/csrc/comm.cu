// Inter-rank transport for time-window sharding (BJ north_star:
// "NCCL send/recv over NVLink carries the one-state halo that L needs
// (M_i x_{i-1}), and NCCL allreduce carries the Krylov inner products").
//
// The hot path needs exactly three collective primitives:
//   exchange     grouped point-to-point copies of contiguous [s][m] window states
//                (halos of L / L^T, chain hand-offs of L_hat^{-1} / L_hat^{-T})
//   allreduce    in-place sum of per-RHS Krylov inner products ([nd][m] doubles)
//   allgather    per-rank window totals of the L_I prefix scan
// Two transports implement them, both stream-ordered (nothing blocks the GPU):
//   NcclComm   one process per GPU; libnccl.so.2 is dlopen'ed (the same soname torch
//              loads, so one NCCL per process) and driven with ncclSend/ncclRecv
//              groups, ncclAllReduce and ncclAllGather on the library stream.
//   LocalComm  G ranks as G host threads of one process (one context each), for
//              driving the sharded path on a single device.  Ranks rendezvous on
//              the host (mutex + condition variable) and hand each other device
//              pointers plus CUDA events: the receiver's stream waits on the
//              sender's "data ready" event and copies; the sender's stream waits on
//              the receiver's "consumed" event before it may overwrite the buffer.
//              Reductions sum the G contributions in rank order, so every rank gets
//              bitwise the same result.  No kernel ever waits on another kernel.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>

#include "internal.h"

namespace wf {

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
#define WF_SYM(field, sym) api.field = (decltype(api.field))dlsym(api.h, sym)
    WF_SYM(GetUniqueId, "ncclGetUniqueId");
    WF_SYM(CommInitRank, "ncclCommInitRank");
    WF_SYM(CommDestroy, "ncclCommDestroy");
    WF_SYM(Send, "ncclSend");
    WF_SYM(Recv, "ncclRecv");
    WF_SYM(AllReduce, "ncclAllReduce");
    WF_SYM(AllGather, "ncclAllGather");
    WF_SYM(GroupStart, "ncclGroupStart");
    WF_SYM(GroupEnd, "ncclGroupEnd");
    WF_SYM(GetErrorString, "ncclGetErrorString");
#undef WF_SYM
  });
  if (!api.h || !api.CommInitRank || !api.Send || !api.AllReduce)
    throw Error{WF4DVAR_ENCCL, "libnccl.so.2 could not be loaded (dlopen)"};
  return api;
}

#define WF_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess)                                                             \
      throw ::wf::Error{WF4DVAR_ENCCL, std::string(#call) + ": " +                     \
                                           (nccl().GetErrorString ? nccl().GetErrorString(r_) : "?")}; \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm(int rank_, int world_, const void *id) {
    rank = rank_;
    world = world_;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    WF_NCCL(nccl().CommInitRank(&comm, world, uid, rank));
  }
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void exchange(const std::vector<P2P> &ops, cudaStream_t st) override {
    if (ops.empty()) return;
    WF_NCCL(nccl().GroupStart());
    for (const P2P &o : ops) {
      if (o.send) WF_NCCL(nccl().Send(o.buf, o.count, ncclFloat64, o.peer, comm, st));
      else WF_NCCL(nccl().Recv(o.buf, o.count, ncclFloat64, o.peer, comm, st));
    }
    WF_NCCL(nccl().GroupEnd());
  }
  void allreduce_sum(double *buf, size_t count, cudaStream_t st) override {
    WF_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm, st));
  }
  void allgather(const double *send, double *recv, size_t count, cudaStream_t st) override {
    WF_NCCL(nccl().AllGather(send, recv, count, ncclFloat64, comm, st));
  }
};
}  // namespace

void nccl_unique_id(void *out128) {
  ncclUniqueId id;
  WF_NCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, sizeof(id));
}

// ------------------------------------------------------------------ in-process group
// out[i] = sum_{g < G} src[g][i], fixed rank order (pointers passed by value)
constexpr int kMaxLocalRanks = 64;
struct RankPtrs { const double *p[kMaxLocalRanks]; };
__global__ void k_sum_ranks(double *out, const RankPtrs src, int G, int64_t count) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double v = 0.0;
  for (int g = 0; g < G; ++g) v += src.p[g][i];
  out[i] = v;
}

struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  // point-to-point: FIFO of posted sends per (src, dst) and of consumed acks
  struct Msg { const double *ptr; size_t count; cudaEvent_t ready; };
  std::map<std::pair<int, int>, std::deque<Msg>> mail;
  std::map<std::pair<int, int>, std::deque<cudaEvent_t>> acks;
  // collectives: generation-indexed rendezvous slots
  struct Coll {
    std::vector<const double *> ptr;
    std::vector<cudaEvent_t> ready, done;
    int posted = 0, finished = 0, left = 0;
  };
  std::map<int64_t, Coll> coll;
  explicit LocalGroup(int w) : world(w) {}
};

namespace {
cudaEvent_t record_new(cudaStream_t st) {
  cudaEvent_t e;
  WF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  WF_CUDA(cudaEventRecord(e, st));
  return e;
}

struct LocalComm : Comm {
  LocalGroup *g;
  int64_t gen = 0;                 // collective generation (same sequence on every rank)
  double *tmp = nullptr;           // reduction result staging
  size_t tmp_cap = 0;
  LocalComm(int rank_, LocalGroup *grp) : g(grp) {
    rank = rank_;
    world = grp->world;
  }
  ~LocalComm() override {
    if (tmp) cudaFree(tmp);
  }
  void exchange(const std::vector<P2P> &ops, cudaStream_t st) override {
    if (ops.empty()) return;
    std::unique_lock<std::mutex> lk(g->mu);
    // 1. post every send (data ready once the stream reaches this point)
    for (const P2P &o : ops)
      if (o.send)
        g->mail[{rank, o.peer}].push_back({(const double *)o.buf, o.count, record_new(st)});
    g->cv.notify_all();
    // 2. receive: wait for the matching post, copy after its ready event
    for (const P2P &o : ops) {
      if (o.send) continue;
      auto &q = g->mail[{o.peer, rank}];
      g->cv.wait(lk, [&] { return !q.empty(); });
      LocalGroup::Msg msg = q.front();
      q.pop_front();
      WF_REQUIRE(msg.count == o.count, WF4DVAR_ENCCL, "local exchange: size mismatch");
      WF_CUDA(cudaStreamWaitEvent(st, msg.ready, 0));
      WF_CUDA(cudaMemcpyAsync(o.buf, msg.ptr, o.count * 8, cudaMemcpyDeviceToDevice, st));
      cudaEventDestroy(msg.ready);   // released once the wait above is satisfied
      g->acks[{o.peer, rank}].push_back(record_new(st));
      g->cv.notify_all();
    }
    // 3. a send buffer may be overwritten only after its receiver copied it
    for (const P2P &o : ops) {
      if (!o.send) continue;
      auto &a = g->acks[{rank, o.peer}];
      g->cv.wait(lk, [&] { return !a.empty(); });
      cudaEvent_t e = a.front();
      a.pop_front();
      WF_CUDA(cudaStreamWaitEvent(st, e, 0));
      cudaEventDestroy(e);
    }
  }

  // post (ptr, ready) for generation gen and wait until all ranks posted
  LocalGroup::Coll &post(std::unique_lock<std::mutex> &lk, const double *ptr, cudaStream_t st) {
    auto &cl = g->coll[gen];
    if (cl.ptr.empty()) {
      cl.ptr.assign(world, nullptr);
      cl.ready.assign(world, nullptr);
      cl.done.assign(world, nullptr);
    }
    cl.ptr[rank] = ptr;
    cl.ready[rank] = record_new(st);
    cl.posted++;
    g->cv.notify_all();
    g->cv.wait(lk, [&] { return cl.posted == world; });
    for (int q = 0; q < world; ++q) WF_CUDA(cudaStreamWaitEvent(st, cl.ready[q], 0));
    return cl;
  }
  // publish "finished reading", wait for everyone, order the stream after all readers
  void finish(std::unique_lock<std::mutex> &lk, LocalGroup::Coll &cl, cudaStream_t st) {
    cl.done[rank] = record_new(st);
    cl.finished++;
    g->cv.notify_all();
    g->cv.wait(lk, [&] { return cl.finished == world; });
    for (int q = 0; q < world; ++q) WF_CUDA(cudaStreamWaitEvent(st, cl.done[q], 0));
    if (++cl.left == world) {
      for (int q = 0; q < world; ++q) {
        cudaEventDestroy(cl.ready[q]);
        cudaEventDestroy(cl.done[q]);
      }
      g->coll.erase(gen);
    }
    ++gen;
  }
  void allreduce_sum(double *buf, size_t count, cudaStream_t st) override {
    if (count > tmp_cap) {
      if (tmp) cudaFree(tmp);
      WF_CUDA(cudaMalloc(&tmp, count * 8));
      tmp_cap = count;
    }
    std::unique_lock<std::mutex> lk(g->mu);
    auto &cl = post(lk, buf, st);
    RankPtrs rp{};
    for (int q = 0; q < world; ++q) rp.p[q] = cl.ptr[q];
    k_sum_ranks<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(tmp, rp, world, (int64_t)count);
    WF_CUDA(cudaGetLastError());
    finish(lk, cl, st);
    WF_CUDA(cudaMemcpyAsync(buf, tmp, count * 8, cudaMemcpyDeviceToDevice, st));
  }
  void allgather(const double *send, double *recv, size_t count, cudaStream_t st) override {
    std::unique_lock<std::mutex> lk(g->mu);
    auto &cl = post(lk, send, st);
    for (int q = 0; q < world; ++q)
      WF_CUDA(cudaMemcpyAsync(recv + (size_t)q * count, cl.ptr[q], count * 8,
                              cudaMemcpyDeviceToDevice, st));
    finish(lk, cl, st);
  }
};
}  // namespace

LocalGroup *local_group_create(int world) {
  WF_REQUIRE(world >= 1 && world <= kMaxLocalRanks, WF4DVAR_EINVAL, "local group: 1 <= world <= 64");
  return new LocalGroup(world);
}
void local_group_destroy(LocalGroup *g) { delete g; }

Comm *make_comm(const wf4dvar_dist &d) {
  // world == 1 with an explicit transport still builds it (single-device check of the
  // transport's calls: a 1-rank communicator, allreduce = copy, no neighbours)
  if (d.world <= 1 && d.transport == WF4DVAR_TRANSPORT_NONE) return nullptr;
  if (d.transport == WF4DVAR_TRANSPORT_NCCL) {
    WF_REQUIRE(d.nccl_id != nullptr, WF4DVAR_EINVAL, "NCCL transport needs nccl_id");
    return new NcclComm(d.rank, d.world, d.nccl_id);
  }
  if (d.transport == WF4DVAR_TRANSPORT_LOCAL) {
    WF_REQUIRE(d.local_group != nullptr, WF4DVAR_EINVAL, "LOCAL transport needs local_group");
    LocalGroup *g = (LocalGroup *)d.local_group;
    WF_REQUIRE(g->world == d.world, WF4DVAR_EINVAL, "local_group world mismatch");
    return new LocalComm(d.rank, g);
  }
  throw Error{WF4DVAR_EINVAL, "world > 1 needs transport NCCL or LOCAL"};
}

}  // namespace wf
