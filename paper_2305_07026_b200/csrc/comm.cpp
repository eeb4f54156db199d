// comm.cpp — NCCL (dlopen) and in-process LOCAL backends of the DABA exchange steps.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

namespace daba {

// ------------------------------------------------------------------ NCCL, resolved at run time
namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
#define LOAD(field, sym)                                                     \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym));          \
  if (!api.field) {                                                          \
    api.err = std::string("libnccl lacks ") + sym;                           \
    return;                                                                  \
  }
    LOAD(GetUniqueId, "ncclGetUniqueId");
    LOAD(CommInitRank, "ncclCommInitRank");
    LOAD(CommDestroy, "ncclCommDestroy");
    LOAD(AllReduce, "ncclAllReduce");
    LOAD(Send, "ncclSend");
    LOAD(Recv, "ncclRecv");
    LOAD(GroupStart, "ncclGroupStart");
    LOAD(GroupEnd, "ncclGroupEnd");
    LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
    api.ok = true;
  });
  return api;
}

std::string nccl_err(const char* what, ncclResult_t r) {
  return std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
}

class NcclComm : public Comm {
 public:
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  std::string allreduce(const double* d_in, double* d_out, int n, cudaStream_t st) override {
    ncclResult_t r = nccl().AllReduce(d_in, d_out, (size_t)n, ncclFloat64, ncclSum, comm, st);
    return r == ncclSuccess ? "" : nccl_err("ncclAllReduce", r);
  }
  std::string exchange(const double* d_send, double* d_recv, const std::vector<PeerSeg>& segs,
                       cudaStream_t st) override {
    ncclResult_t r = nccl().GroupStart();
    if (r != ncclSuccess) return nccl_err("ncclGroupStart", r);
    for (const PeerSeg& s : segs) {
      if (s.send_cnt > 0) {
        r = nccl().Send(d_send + s.send_off, (size_t)s.send_cnt, ncclFloat64, s.rank, comm, st);
        if (r != ncclSuccess) break;
      }
      if (s.recv_cnt > 0) {
        r = nccl().Recv(d_recv + s.recv_off, (size_t)s.recv_cnt, ncclFloat64, s.rank, comm, st);
        if (r != ncclSuccess) break;
      }
    }
    ncclResult_t r2 = nccl().GroupEnd();
    if (r != ncclSuccess) return nccl_err("ncclSend/Recv", r);
    return r2 == ncclSuccess ? "" : nccl_err("ncclGroupEnd", r2);
  }
  std::string allreduce_exchange(const double* d_in, double* d_out, int n, const double* d_send, double* d_recv,
                                 const std::vector<PeerSeg>& segs, cudaStream_t st) override {
    ncclResult_t r = nccl().GroupStart();
    if (r != ncclSuccess) return nccl_err("ncclGroupStart", r);
    r = nccl().AllReduce(d_in, d_out, (size_t)n, ncclFloat64, ncclSum, comm, st);
    for (const PeerSeg& s : segs) {
      if (r != ncclSuccess) break;
      if (s.send_cnt > 0) r = nccl().Send(d_send + s.send_off, (size_t)s.send_cnt, ncclFloat64, s.rank, comm, st);
      if (r == ncclSuccess && s.recv_cnt > 0)
        r = nccl().Recv(d_recv + s.recv_off, (size_t)s.recv_cnt, ncclFloat64, s.rank, comm, st);
    }
    ncclResult_t r2 = nccl().GroupEnd();
    if (r != ncclSuccess) return nccl_err("ncclAllReduce/Send/Recv", r);
    return r2 == ncclSuccess ? "" : nccl_err("ncclGroupEnd", r2);
  }
  bool capturable() const override { return true; }
};

// ------------------------------------------------------------------ LOCAL: ranks = threads of one process
struct Hub {
  int nranks;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  std::vector<std::vector<double>> red;                 // allreduce slots
  std::vector<const double*> send_ptr;                  // exchange: each rank's send buffer
  std::vector<std::vector<PeerSeg>> segs;               // and its segments
  explicit Hub(int n) : nranks(n), red((size_t)n), send_ptr((size_t)n, nullptr), segs((size_t)n) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

// NONE (measurement only): one rank's shard without peers.  The allreduce is a local copy (so the iteration's
// kernels run unchanged), the exchange moves nothing.
class NoneComm : public Comm {
 public:
  std::string allreduce(const double* d_in, double* d_out, int n, cudaStream_t st) override {
    return cudaMemcpyAsync(d_out, d_in, sizeof(double) * n, cudaMemcpyDeviceToDevice, st) == cudaSuccess
               ? ""
               : "NONE allreduce: copy failed";
  }
  std::string exchange(const double*, double*, const std::vector<PeerSeg>&, cudaStream_t) override { return ""; }
  bool capturable() const override { return true; }
};

std::mutex g_hub_mu;
std::map<std::string, std::weak_ptr<Hub>> g_hubs;

class LocalComm : public Comm {
 public:
  std::shared_ptr<Hub> hub;
  int rank;
  std::string allreduce(const double* d_in, double* d_out, int n, cudaStream_t st) override {
    std::vector<double> mine((size_t)n);
    if (cudaMemcpyAsync(mine.data(), d_in, sizeof(double) * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return "LOCAL allreduce: D2H failed";
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      hub->red[(size_t)rank] = mine;
    }
    hub->barrier();
    std::vector<double> sum((size_t)n, 0.0);
    for (int r = 0; r < hub->nranks; ++r)  // fixed rank order: deterministic
      for (int k = 0; k < n; ++k) sum[(size_t)k] += hub->red[(size_t)r][(size_t)k];
    hub->barrier();
    if (cudaMemcpyAsync(d_out, sum.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return "LOCAL allreduce: H2D failed";
    return "";
  }
  std::string exchange(const double* d_send, double* d_recv, const std::vector<PeerSeg>& segs,
                       cudaStream_t st) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) return "LOCAL exchange: sync failed";
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      hub->send_ptr[(size_t)rank] = d_send;
      hub->segs[(size_t)rank] = segs;
    }
    hub->barrier();
    std::string err;
    for (const PeerSeg& s : segs) {
      if (s.recv_cnt == 0) continue;
      const PeerSeg* src = nullptr;
      for (const PeerSeg& q : hub->segs[(size_t)s.rank])
        if (q.rank == rank) src = &q;
      if (!src || src->send_cnt != s.recv_cnt) {
        err = "LOCAL exchange: peer segment mismatch";
        break;
      }
      if (cudaMemcpyAsync(d_recv + s.recv_off, hub->send_ptr[(size_t)s.rank] + src->send_off,
                          sizeof(double) * (size_t)s.recv_cnt, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
        err = "LOCAL exchange: copy failed";
        break;
      }
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && err.empty()) err = "LOCAL exchange: sync failed";
    hub->barrier();
    return err;
  }
  bool capturable() const override { return false; }
};

}  // namespace

std::string nccl_unique_id(void* id_out) {
  NcclApi& api = nccl();
  if (!api.ok) return api.err;
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_err("ncclGetUniqueId", r);
  std::memcpy(id_out, &id, sizeof id);
  return "";
}

Comm* make_comm(int kind, const void* id, int rank, int nranks, std::string* err) {
  if (kind == 2) return new NoneComm();
  if (kind == 1) {
    std::string key(static_cast<const char*>(id), 128);
    std::shared_ptr<Hub> hub;
    {
      std::lock_guard<std::mutex> lk(g_hub_mu);
      auto it = g_hubs.find(key);
      if (it != g_hubs.end()) hub = it->second.lock();
      if (!hub) {
        hub = std::make_shared<Hub>(nranks);
        g_hubs[key] = hub;
      }
    }
    if (hub->nranks != nranks) {
      *err = "LOCAL hub: nranks mismatch";
      return nullptr;
    }
    auto* c = new LocalComm();
    c->hub = hub;
    c->rank = rank;
    return c;
  }
  NcclApi& api = nccl();
  if (!api.ok) {
    *err = api.err;
    return nullptr;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  auto* c = new NcclComm();
  ncclResult_t r = api.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    *err = nccl_err("ncclCommInitRank", r);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

}  // namespace daba
