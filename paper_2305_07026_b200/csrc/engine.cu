// engine.cu — per-rank DABA engine behind the C-ABI of include/daba.h.
//
// Host work happens only in daba_create / daba_set_state_native / daba_get_state: shard planning, layout
// conversion, uploads.  daba_iterate enqueues device work only (optionally replaying a captured CUDA graph);
// the restart decision, the role rotation and the schedule live on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/daba.h"
#include "comm.h"
#include "kernels.h"
#include "shard.h"

using namespace daba;

thread_local std::string g_create_err = "";  // why this thread's last daba_create failed
thread_local int g_bail_line = 0;

struct daba_ctx {
  std::string err;
  int device = 0, rank = 0, nranks = 1;
  cudaStream_t stream = nullptr, side = nullptr;  // side: the k_cam_solve branch of an iteration
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fork0 = nullptr, ev_join0 = nullptr;
  int num_sms = 148;
  bool own_stream = false;
  daba_options opt{};
  daba_loss loss{};
  ShardPlan plan;
  std::unique_ptr<Comm> comm;
  std::vector<void*> allocs;
  bool pooled = false;  // allocs come from context_pool (freed stream-ordered)
  size_t dev_bytes = 0;
  IterParams P{};
  int64_t host_k = 0;
  double* d_metric = nullptr;  // 4 doubles, daba_pixel_error (allocated on first use)
  // halo exchange
  std::vector<PeerSeg> segs;
  int32_t *d_send_cam = nullptr, *d_send_pt = nullptr, *d_recv_cam = nullptr, *d_recv_pt = nullptr;
  int64_t *d_send_cam_off = nullptr, *d_send_pt_off = nullptr, *d_recv_cam_off = nullptr, *d_recv_pt_off = nullptr;
  int32_t n_send_cam = 0, n_send_pt = 0, n_recv_cam = 0, n_recv_pt = 0;
  double *d_sendbuf = nullptr, *d_recvbuf = nullptr;
  // graph
  cudaGraphExec_t graph = nullptr;
  bool graph_failed = false;
  int launches_per_iter = 0;
  // parallel graph branches (A/B switches, environment at create): boundary records beside the camera pass
  // (DABA_FORK0=1; measured slower at 8 ranks: 0.272 vs 0.258 ms), the solve beside the point pass
  // (DABA_FORK1=0 disables)
  bool fork0 = false, fork1 = true;
  // profiling
  std::vector<std::string> knames;
  std::vector<double> kms;
  std::vector<int64_t> klaunches;
  struct Pending {
    int name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
};

namespace {

// Split [0, n) over the host's cores (create-time setup loops only; the iteration itself never runs here).
template <class F>
void parallel_for(int64_t n, F&& f) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < (1 << 16) || hw == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (unsigned t = 0; t < hw; ++t) th.emplace_back([&, t] { f(n * t / hw, n * (t + 1) / hw); });
  for (auto& x : th) x.join();
}

// Integer tuning knob from the environment (create time only), else the default.
int64_t env_int(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return (int64_t)std::atoll(v);
}

// Create-time phase timer (DABA_TIMING=1 prints the host cost of each phase of daba_create to stderr).
struct PhaseTimer {
  bool on = std::getenv("DABA_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    const cudaError_t e = cudaPeekAtLastError();
    fprintf(stderr, "daba_create %-28s %8.1f ms%s%s\n", what, std::chrono::duration<double, std::milli>(n - t).count(),
            e ? "  pending CUDA error: " : "", e ? cudaGetErrorString(e) : "");
    t = n;
  }
};

int fail(daba_ctx* c, int code, const std::string& m) {
  if (c) c->err = m;
  return code;
}

#define CUDA_OR(ctx, x)                                                                          \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return fail(ctx, DABA_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Device memory of the contexts comes from a process-wide stream-ordered pool per device that keeps what
// destroyed contexts free (release threshold = max): a later daba_create in the same process reuses mapped
// memory instead of paying the driver's page mapping again (cudaMalloc of the ~1 GB of Final-13682 state measured
// 4-55 ms right after a previous context's cudaFree).  DABA_POOL=0: plain cudaMalloc / cudaFree.
cudaMemPool_t context_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  static bool tried[64] = {};
  if (device < 0 || device >= 64 || env_int("DABA_POOL", 1) == 0) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!tried[device]) {
    tried[device] = true;
    cudaMemPoolProps pr{};
    pr.allocType = cudaMemAllocationTypePinned;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = device;
    if (cudaMemPoolCreate(&pools[device], &pr) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep);
    } else {
      pools[device] = nullptr;
      cudaGetLastError();
    }
  }
  return pools[device];
}

template <class T>
int dalloc(daba_ctx* c, T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  cudaMemPool_t pool = context_pool(c->device);
  cudaError_t e = pool ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), n * sizeof(T), pool, c->stream)
                       : cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
  if (pool) c->pooled = true;
  if (e != cudaSuccess) return fail(c, e == cudaErrorMemoryAllocation ? DABA_E_OOM : DABA_E_CUDA,
                                    std::string("cudaMalloc: ") + cudaGetErrorString(e));
  c->allocs.push_back(*p);
  c->dev_bytes += n * sizeof(T);
  return DABA_OK;
}

// Release one dalloc'd buffer before destroy (create-time buffers whose job is done).
void dfree(daba_ctx* c, void* p, size_t bytes) {
  if (!p) return;
  auto it = std::find(c->allocs.begin(), c->allocs.end(), p);
  if (it == c->allocs.end()) return;
  c->allocs.erase(it);
  c->dev_bytes -= bytes;
  if (c->pooled)
    cudaFreeAsync(p, c->stream);
  else
    cudaFree(p);
}

// Host -> device copy on the context's stream.  Small or page-locked sources go directly; large pageable ones
// through a process-wide page-locked staging buffer (two 32 MB halves: the host threads fill one half while
// the copy engine drains the other).  Returns once the source may be reused.
// process-wide page-locked staging buffer of two 32 MB halves (allocated on first use; null if that failed)
constexpr size_t kStageHalf = 32u << 20;
std::mutex g_stage_mu;
char* g_stage = nullptr;
cudaEvent_t g_stage_ev[2] = {nullptr, nullptr};
bool g_stage_tried = false;

char* stage_buffer() {  // call with g_stage_mu held
  if (!g_stage_tried) {
    g_stage_tried = true;
    if (cudaMallocHost(&g_stage, 2 * kStageHalf) != cudaSuccess) {
      g_stage = nullptr;
      cudaGetLastError();
    } else {
      cudaEventCreateWithFlags(&g_stage_ev[0], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g_stage_ev[1], cudaEventDisableTiming);
    }
  }
  return g_stage;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();  // a pageable pointer may leave an error behind on some drivers
  return pinned;
}

cudaError_t h2d(daba_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  if (bytes < (8u << 20) || is_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream);
  std::lock_guard<std::mutex> lk(g_stage_mu);
  char* stage = stage_buffer();
  if (!stage) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream);
  bool used[2] = {false, false};
  for (size_t off = 0, h = 0; off < bytes; off += kStageHalf, h ^= 1) {
    const size_t n = std::min(kStageHalf, bytes - off);
    if (used[h]) cudaEventSynchronize(g_stage_ev[h]);
    char* buf = stage + h * kStageHalf;
    const char* s = static_cast<const char*>(src) + off;
    parallel_for((int64_t)n, [&](int64_t a, int64_t b) { std::memcpy(buf + a, s + a, (size_t)(b - a)); });
    cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf, n, cudaMemcpyHostToDevice, c->stream);
    if (e != cudaSuccess) return e;
    cudaEventRecord(g_stage_ev[h], c->stream);
    used[h] = true;
  }
  for (int h = 0; h < 2; ++h)
    if (used[h]) cudaEventSynchronize(g_stage_ev[h]);  // the staging buffer is free for the next caller
  return cudaSuccess;
}

// Device -> host, blocking: large pageable destinations through the staging halves (the copy engine fills one
// half while host threads empty the other) instead of the driver's single-threaded pageable path.
cudaError_t d2h(daba_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  if (bytes < (8u << 20) || is_pinned(dst)) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream);
    return e != cudaSuccess ? e : cudaStreamSynchronize(c->stream);
  }
  std::lock_guard<std::mutex> lk(g_stage_mu);
  char* stage = stage_buffer();
  if (!stage) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream);
    return e != cudaSuccess ? e : cudaStreamSynchronize(c->stream);
  }
  const size_t nchunk = (bytes + kStageHalf - 1) / kStageHalf;
  auto issue = [&](size_t q) {
    const size_t off = q * kStageHalf, n = std::min(kStageHalf, bytes - off);
    cudaError_t e = cudaMemcpyAsync(stage + (q & 1) * kStageHalf, static_cast<const char*>(src) + off, n,
                                    cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaEventRecord(g_stage_ev[q & 1], c->stream);
    return e;
  };
  cudaError_t e = issue(0);
  for (size_t q = 0; q < nchunk && e == cudaSuccess; ++q) {
    if (q + 1 < nchunk && (e = issue(q + 1)) != cudaSuccess) break;
    if ((e = cudaEventSynchronize(g_stage_ev[q & 1])) != cudaSuccess) break;
    const size_t off = q * kStageHalf, n = std::min(kStageHalf, bytes - off);
    const char* buf = stage + (q & 1) * kStageHalf;
    char* d = static_cast<char*>(dst) + off;
    parallel_for((int64_t)n, [&](int64_t a, int64_t b) { std::memcpy(d + a, buf + a, (size_t)(b - a)); });
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return e;
}

template <class T, class A>
int upload(daba_ctx* c, T** p, const std::vector<T, A>& h) {
  int rc = dalloc(c, p, h.size());
  if (rc) return rc;
  CUDA_OR(c, h2d(c, *p, h.data(), h.size() * sizeof(T)));
  return DABA_OK;
}

int name_index(daba_ctx* c, const char* name) {
  for (size_t i = 0; i < c->knames.size(); ++i)
    if (c->knames[i] == name) return (int)i;
  c->knames.push_back(name);
  c->kms.push_back(0.0);
  c->klaunches.push_back(0);
  return (int)c->knames.size() - 1;
}

cudaEvent_t take_event(daba_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Run one launcher, bracketed by events in profile mode.
template <class F>
int timed(daba_ctx* c, const char* name, F&& fn) {
  if (!c->opt.profile) return fn();
  const int id = name_index(c, name);
  cudaEvent_t a = take_event(c), b = take_event(c);
  cudaEventRecord(a, c->stream);
  const int n = fn();
  cudaEventRecord(b, c->stream);
  if (n == 0) {  // nothing launched: no entry
    c->event_pool.push_back(a);
    c->event_pool.push_back(b);
    return 0;
  }
  c->pending.push_back({id, a, b});
  c->klaunches[(size_t)id] += n;
  return n;
}

void collect_times(daba_ctx* c) {
  for (auto& p : c->pending) {
    float ms = 0;
    cudaEventSynchronize(p.b);
    cudaEventElapsedTime(&ms, p.a, p.b);
    c->kms[(size_t)p.name] += ms;
    c->event_pool.push_back(p.a);
    c->event_pool.push_back(p.b);
  }
  c->pending.clear();
}

// Enqueue one iteration of Algorithm 1.  With a communicator and the global restart test, the solves write both
// candidates of every boundary variable into the send buffer, which is exchanged in the same NCCL group as the
// allreduce of the restart sums (the two transfers overlap); k_unpack then takes the decision from the
// allreduced sums, keeps the selected candidate and commits the decision.  With the per-device test the rank
// decides in the solves' last block and sends x^{k+1} (k_pack); the allreduce only feeds the trace.
int enqueue_iteration(daba_ctx* c, int* launches) {
  const IterParams& P = c->P;
  int n = 0;
  if (!c->opt.profile && c->fork0 && (P.n_boundary > 0 || P.n_inter_blocks > 0)) {
    // the boundary records and the inter-device terms only read x^k, x-bar^k and the halo: a parallel branch
    // beside the camera pass
    CUDA_OR(c, cudaEventRecord(c->ev_fork0, c->stream));
    CUDA_OR(c, cudaStreamWaitEvent(c->side, c->ev_fork0, 0));
    n += launch_pt_pass(P, c->side);
    n += launch_inter(P, c->side);
    CUDA_OR(c, cudaEventRecord(c->ev_join0, c->side));
    n += launch_cam_pass(P, c->stream);
    CUDA_OR(c, cudaStreamWaitEvent(c->stream, c->ev_join0, 0));
  } else {
    n += timed(c, "k_cam_pass", [&] { return launch_cam_pass(P, c->stream); });
    n += timed(c, "k_pt_boundary", [&] { return launch_pt_pass(P, c->stream); });
    n += timed(c, "k_inter", [&] { return launch_inter(P, c->stream); });
  }
  // k_cam_solve and k_pt_sum are independent: parallel graph branches (the solve hides behind the point pass;
  // measured 1.3451 -> 1.3423 ms at 13.7K cameras, and it is what keeps the solve off the critical path at 8
  // ranks).  Profiling always serialises so events bracket one kernel; DABA_FORK1=0 serialises.
  if (c->opt.profile || !c->fork1) {
    n += timed(c, "k_cam_solve", [&] { return launch_cam_solve(P, c->stream); });
    n += timed(c, "k_pt_sum", [&] { return launch_pt_sum(P, c->stream); });
  } else {
    // k_cam_solve and k_pt_sum are independent: fork a second stream (captured as parallel graph branches)
    CUDA_OR(c, cudaEventRecord(c->ev_fork, c->stream));
    CUDA_OR(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    n += launch_cam_solve(P, c->side);
    CUDA_OR(c, cudaEventRecord(c->ev_join, c->side));
    n += launch_pt_sum(P, c->stream);
    CUDA_OR(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  }
  if (c->comm) {
    const bool halo = !c->segs.empty();
    const bool dev = P.restart_scope == 1;
    if (halo && !P.sendbuf)  // (global test: the solves already wrote the send buffer)
      n += timed(c, "k_pack", [&] {
        return launch_pack(P, c->d_send_cam, c->d_send_cam_off, c->n_send_cam, c->d_send_pt, c->d_send_pt_off,
                           c->n_send_pt, c->d_sendbuf, dev ? 1 : 0, c->stream);
      });
    std::string e = c->comm->allreduce_exchange(P.local, P.global, kGlobalCols, c->d_sendbuf, c->d_recvbuf,
                                                halo ? c->segs : std::vector<PeerSeg>(), c->stream);
    if (!e.empty()) return fail(c, DABA_E_NCCL, e);
    // the global decision is taken inside k_unpack when there is one; otherwise by k_select
    const bool unpack = c->n_recv_cam + c->n_recv_pt > 0;
    if (dev)
      n += timed(c, "k_trace_post", [&] { return launch_trace_post(P, c->stream); });
    else if (!unpack)
      n += timed(c, "k_select", [&] { return launch_select(P, c->stream); });
    if (unpack)
      n += timed(c, "k_unpack", [&] {
        return launch_unpack(P, c->d_recv_cam, c->d_recv_cam_off, c->n_recv_cam, c->d_recv_pt, c->d_recv_pt_off,
                             c->n_recv_pt, c->d_recvbuf, dev ? 0 : 1, c->stream);
      });
  }
  *launches += n;
  CUDA_OR(c, cudaGetLastError());
  return DABA_OK;
}

int compute_objective(daba_ctx* c, double* F, double* ndeg) {
  launch_objective(c->P, c->stream);
  if (c->comm) {
    std::string e = c->comm->allreduce(c->P.local, c->P.global, kGlobalCols, c->stream);
    if (!e.empty()) return fail(c, DABA_E_NCCL, e);
  }
  double g[kGlobalCols];
  CUDA_OR(c, cudaMemcpyAsync(g, c->comm ? c->P.global : c->P.local, sizeof g, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR(c, cudaStreamSynchronize(c->stream));
  *F = g[0];
  if (ndeg) *ndeg = g[7];
  return DABA_OK;
}

// Upload global native states into the local role buffers `rk` (x^k) and `rkm1` (x^{k-1}).
int upload_states(daba_ctx* c, const double* cams_k, const double* pts_k, const double* cams_km1,
                  const double* pts_km1, int rk, int rkm1) {
  const ShardPlan& S = c->plan;
  int h_roles[4];
  CUDA_OR(c, cudaMemcpyAsync(h_roles, c->P.roles, sizeof h_roles, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR(c, cudaStreamSynchronize(c->stream));
  // light plan (identity point numbering, one rank): the caller's xyz go to the device as they are (through the
  // record staging buffer, free outside iterations) and are widened to 32 B records there
  const size_t np = S.pt_g.size();
  const bool direct = S.point_side_deferred && (int64_t)np == S.N && c->P.staging &&
                      3 * np <= 8 * (size_t)c->P.n_records;
  hvec<double> hc(S.cam_g.size() * kCamStride), hp(direct ? 0 : np * 4);
  for (int pass = 0; pass < 2; ++pass) {
    const double* gc = pass ? cams_km1 : cams_k;
    const double* gp = pass ? pts_km1 : pts_k;
    if (pass == 1 && cams_km1 == cams_k && pts_km1 == pts_k) {  // x^{k-1} = x^k (create): a device copy
      CUDA_OR(c, cudaMemcpyAsync(c->P.cams[h_roles[rkm1]], c->P.cams[h_roles[rk]], hc.size() * sizeof(double),
                                 cudaMemcpyDeviceToDevice, c->stream));
      CUDA_OR(c, cudaMemcpyAsync(c->P.pts[h_roles[rkm1]], c->P.pts[h_roles[rk]], np * 4 * sizeof(double),
                                 cudaMemcpyDeviceToDevice, c->stream));
      break;
    }
    parallel_for((int64_t)S.cam_g.size(), [&](int64_t a, int64_t b) {
      for (int64_t li = a; li < b; ++li) {
        std::memcpy(&hc[(size_t)li * kCamStride], gc + 15 * (size_t)S.cam_g[(size_t)li], 15 * sizeof(double));
        hc[(size_t)li * kCamStride + 15] = 0.0;
      }
    });
    const int role = pass ? rkm1 : rk;
    if (direct) {
      CUDA_OR(c, h2d(c, c->P.staging, gp, 3 * np * sizeof(double)));
      launch_xyz_pts(c->P.staging, c->P.pts[h_roles[role]], (int32_t)np, c->stream);
      CUDA_OR(c, cudaGetLastError());
    } else {
      parallel_for((int64_t)np, [&](int64_t a, int64_t b) {
        for (int64_t lj = a; lj < b; ++lj) {
          for (int k = 0; k < 3; ++k) hp[(size_t)lj * 4 + k] = gp[3 * (size_t)S.pt_g[(size_t)lj] + k];
          hp[(size_t)lj * 4 + 3] = 0.0;
        }
      });
      CUDA_OR(c, h2d(c, c->P.pts[h_roles[role]], hp.data(), hp.size() * sizeof(double)));
    }
    CUDA_OR(c, h2d(c, c->P.cams[h_roles[role]], hc.data(), hc.size() * sizeof(double)));
    CUDA_OR(c, cudaStreamSynchronize(c->stream));  // the host buffers are refilled by the next pass
  }
  return DABA_OK;
}

}  // namespace

namespace daba {
// BAL (angle-axis R_w2c, t_w2c, f, k1, k2) -> native (R camera->world, centre t, d = (f, f k1, f k2)).
void bal_to_native(const double* b, double* c) {
  const double wx = b[0], wy = b[1], wz = b[2];
  const double th2 = wx * wx + wy * wy + wz * wz;
  double A, B;
  if (th2 < 1e-16) {
    A = 1.0 - th2 / 6.0;
    B = 0.5 - th2 / 24.0;
  } else {
    const double th = std::sqrt(th2);
    A = std::sin(th) / th;
    const double h = std::sin(0.5 * th);
    B = 2.0 * h * h / th2;
  }
  // Q = R_w2c = I + A [w]x + B [w]x^2
  const double Q[9] = {1.0 + B * (wx * wx - th2), -A * wz + B * wx * wy,     A * wy + B * wx * wz,
                       A * wz + B * wx * wy,      1.0 + B * (wy * wy - th2), -A * wx + B * wy * wz,
                       -A * wy + B * wx * wz,     A * wx + B * wy * wz,      1.0 + B * (wz * wz - th2)};
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) c[3 * r + k] = Q[3 * k + r];  // R = Q^T
  for (int r = 0; r < 3; ++r) c[9 + r] = -(c[3 * r] * b[3] + c[3 * r + 1] * b[4] + c[3 * r + 2] * b[5]);  // t = -R t_w2c
  c[12] = b[6];
  c[13] = b[6] * b[7];
  c[14] = b[6] * b[8];
  c[15] = 0.0;
}

// native -> BAL via the quaternion of R_w2c = R^T (robust for every angle)
void native_to_bal(const double* c, double* b) {
  const double Q[9] = {c[0], c[3], c[6], c[1], c[4], c[7], c[2], c[5], c[8]};
  double w, x, y, z;
  const double tr = Q[0] + Q[4] + Q[8];
  if (tr > Q[0] && tr > Q[4] && tr > Q[8]) {
    const double s = 2.0 * std::sqrt(1.0 + tr);
    w = 0.25 * s; x = (Q[7] - Q[5]) / s; y = (Q[2] - Q[6]) / s; z = (Q[3] - Q[1]) / s;
  } else if (Q[0] > Q[4] && Q[0] > Q[8]) {
    const double s = 2.0 * std::sqrt(1.0 + Q[0] - Q[4] - Q[8]);
    w = (Q[7] - Q[5]) / s; x = 0.25 * s; y = (Q[1] + Q[3]) / s; z = (Q[2] + Q[6]) / s;
  } else if (Q[4] > Q[8]) {
    const double s = 2.0 * std::sqrt(1.0 + Q[4] - Q[0] - Q[8]);
    w = (Q[2] - Q[6]) / s; x = (Q[1] + Q[3]) / s; y = 0.25 * s; z = (Q[5] + Q[7]) / s;
  } else {
    const double s = 2.0 * std::sqrt(1.0 + Q[8] - Q[0] - Q[4]);
    w = (Q[3] - Q[1]) / s; x = (Q[2] + Q[6]) / s; y = (Q[5] + Q[7]) / s; z = 0.25 * s;
  }
  if (w < 0) { w = -w; x = -x; y = -y; z = -z; }
  const double vn = std::sqrt(x * x + y * y + z * z);
  const double ang = 2.0 * std::atan2(vn, w);
  const double f = vn > 0 ? ang / vn : 0.0;
  b[0] = x * f; b[1] = y * f; b[2] = z * f;
  for (int k = 0; k < 3; ++k) b[3 + k] = -(Q[3 * k] * c[9] + Q[3 * k + 1] * c[10] + Q[3 * k + 2] * c[11]);
  b[6] = c[12];
  b[7] = c[13] / c[12];
  b[8] = c[14] / c[12];
}
}  // namespace daba

// ====================================================================== C-ABI
extern "C" int daba_bal_to_native(const double* cameras_bal, int64_t M, double* cameras_native) {
  if (M < 0 || (M > 0 && (!cameras_bal || !cameras_native))) return DABA_E_INVALID_ARG;
  for (int64_t i = 0; i < M; ++i) {
    double tmp[16];
    daba::bal_to_native(cameras_bal + 9 * i, tmp);
    std::memcpy(cameras_native + 15 * i, tmp, 15 * sizeof(double));
  }
  return DABA_OK;
}

extern "C" void daba_default_options(daba_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->xi = 1e-4;
  o->eta = 0.1;
  o->lm_mu0 = 1e-3;
  o->lm_mu_up = 10.0;
  o->eps = 1e-8;
  o->lm_max_trials = 5;
  o->accelerate = 1;
  o->comm = DABA_COMM_NCCL;
  o->use_graph = 1;
  o->profile = 0;
  o->stream = nullptr;
}

extern "C" int daba_comm_id(void* id_out) {
  if (!id_out) return DABA_E_INVALID_ARG;
  return nccl_unique_id(id_out).empty() ? DABA_OK : DABA_E_NCCL;
}

extern "C" int daba_create(const double* cameras, int64_t M, const double* points, int64_t N, const int32_t* obs_cam,
                           const int32_t* obs_pt, const double* obs_uv, int64_t K, daba_loss loss,
                           const int32_t* cam_owner, const int32_t* pt_owner, int rank, int nranks,
                           const void* comm_id, int cuda_device, const daba_options* opt, daba_ctx** out) {
  if (!out) return DABA_E_INVALID_ARG;
  *out = nullptr;
  std::unique_ptr<daba_ctx> c(new (std::nothrow) daba_ctx());
  if (!c) return DABA_E_OOM;
  daba_ctx* C = c.get();
  if (opt)
    C->opt = *opt;
  else
    daba_default_options(&C->opt);
  const daba_options& o = C->opt;
  if (M < 0 || N < 0 || K < 0 || (M > 0 && !cameras) || (N > 0 && !points) || (K > 0 && (!obs_cam || !obs_pt || !obs_uv)))
    return DABA_E_INVALID_ARG;
  if (!(loss.scale > 0) || loss.kind < DABA_LOSS_TRIVIAL || loss.kind > DABA_LOSS_CAUCHY) return DABA_E_INVALID_ARG;
  if (!(o.xi > 0) || !(o.eta > 0 && o.eta <= 1) || !(o.lm_mu0 > 0) || !(o.lm_mu_up >= 1) || !(o.eps >= 0) ||
      o.lm_max_trials < 1 || o.lm_max_trials > 8 || o.restart_scope < 0 || o.restart_scope > 1)
    return DABA_E_INVALID_ARG;
  if (o.comm < DABA_COMM_NCCL || o.comm > DABA_COMM_NONE) return DABA_E_INVALID_ARG;
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !comm_id && o.comm != DABA_COMM_NONE))
    return DABA_E_INVALID_ARG;
  C->loss = loss;
  C->rank = rank;
  C->nranks = nranks;
  C->device = cuda_device;
  C->fork0 = env_int("DABA_FORK0", 0) == 1;
  C->fork1 = std::getenv("DABA_FORK1") == nullptr || std::atoi(std::getenv("DABA_FORK1")) != 0;
  PhaseTimer timer;
  // point numbering for locality (shard.h); DABA_POINT_ORDER = 0 off, 1 automatic (default), 2 always
  const int64_t point_order = env_int("DABA_POINT_ORDER", 1);
  const int32_t point_far = (int32_t)env_int("DABA_POINT_FAR", 1024);  // "far apart" in camera ids
  // one rank with input sorted by (camera, point): a light host plan, the point side built on the device
  const bool defer = nranks == 1 && point_order != 2 && env_int("DABA_DEVICE_PLAN", 1) != 0;
  // device, stream and communicator first: with one rank the observations go to the device anyway, and their
  // validation (indices in range, sorted by (camera, point), each camera's offset) runs there
  if (cudaSetDevice(cuda_device) != cudaSuccess) return DABA_E_CUDA;
  if (o.stream) {
    C->stream = static_cast<cudaStream_t>(o.stream);
  } else {
    if (cudaStreamCreateWithFlags(&C->stream, cudaStreamNonBlocking) != cudaSuccess) return DABA_E_CUDA;
    C->own_stream = true;
  }
  cudaDeviceGetAttribute(&C->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  if (cudaStreamCreateWithFlags(&C->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&C->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&C->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&C->ev_fork0, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&C->ev_join0, cudaEventDisableTiming) != cudaSuccess) {
    daba_destroy(c.release());
    return DABA_E_CUDA;
  }
  if (nranks > 1 || comm_id || o.comm == DABA_COMM_NONE) {  // a single rank with a comm id still routes its
                                                            // sums through the communicator
    std::string ce;
    C->comm.reset(make_comm(o.comm, comm_id, rank, nranks, &ce));
    if (!C->comm) {
      fprintf(stderr, "daba_create: %s\n", ce.c_str());
      daba_destroy(c.release());
      return DABA_E_NCCL;
    }
  }
  int rc = DABA_OK;
  // a failed create leaves its reason for daba_last_error(NULL) (this thread)
  auto bail = [&](int code) {
    std::string why = C->err;
    const cudaError_t ce = cudaGetLastError();
    if (why.empty()) why = code == DABA_E_CUDA ? std::string("CUDA: ") + cudaGetErrorString(ce) : "daba_create failed";
    why += " (engine.cu:" + std::to_string(g_bail_line) + ")";
    daba_destroy(c.release());
    g_create_err = why;
    return code;
  };
  int32_t* d_opt = nullptr;
  bool pre = false;  // a light plan from the device check; the observations are already on the device
  if (defer && !cam_owner && !pt_owner && K > 0 && M > 0 && env_int("DABA_DEVICE_VALIDATE", 1) != 0 &&
      ((4 * (size_t)K + 255) / 256 * 256 + 8 * ((size_t)M + 1) + 1024 <= 64 * (size_t)K)) {
    IterParams& Q = C->P;
    Q.n_records = std::max<int64_t>(K, 1);
    if ((rc = dalloc(C, &Q.staging, 8 * (size_t)Q.n_records)) || (rc = dalloc(C, &d_opt, (size_t)Q.n_records)))
      return g_bail_line = __LINE__, bail(rc);
    int32_t* d_ocam = reinterpret_cast<int32_t*>(Q.staging);
    if (h2d(C, d_opt, obs_pt, sizeof(int32_t) * (size_t)K) != cudaSuccess ||
        h2d(C, d_ocam, obs_cam, sizeof(int32_t) * (size_t)K) != cudaSuccess)
      return g_bail_line = __LINE__, bail(DABA_E_CUDA);
    std::vector<int64_t> cptr((size_t)M + 1);
    int64_t bad = K;
    bool sorted = false;
    if (validate_sorted_device(d_ocam, d_opt, K, M, N,
                               reinterpret_cast<char*>(Q.staging) + (4 * (size_t)K + 255) / 256 * 256, &bad, &sorted,
                               cptr.data(), C->stream) != 0)
      return g_bail_line = __LINE__, bail(DABA_E_CUDA);
    if (bad < K) {
      fail(C, DABA_E_INVALID_ARG, "observation " + std::to_string(bad) + " has an index out of range");
      return g_bail_line = __LINE__, bail(DABA_E_INVALID_ARG);
    }
    if (sorted) {
      plan_light(M, N, K, std::move(cptr), &C->plan);
      pre = true;
    } else {  // the host plan sorts and checks for duplicates
      dfree(C, Q.staging, 64 * (size_t)Q.n_records);
      dfree(C, d_opt, 4 * (size_t)Q.n_records);
      Q.staging = nullptr;
      d_opt = nullptr;
    }
    timer.mark("device validation");
  }
  if (!pre) {
    std::string e = plan_shard(M, N, K, obs_cam, obs_pt, cam_owner, pt_owner, rank, nranks, &C->plan, defer);
    if (!e.empty()) {
      fail(C, DABA_E_INVALID_ARG, e);
      return g_bail_line = __LINE__, bail(DABA_E_INVALID_ARG);
    }
    timer.mark("plan_shard");
    if (!C->plan.point_side_deferred && point_order != 0)
      order_owned_points(&C->plan, obs_cam, point_order == 2, point_far);
    timer.mark("point order");
  }
  // native cameras (Assumption 2 at x^0, is checked on the device by the first objective evaluation)
  std::vector<double> nat((size_t)M * 15);
  for (int64_t i = 0; i < M; ++i) {
    double tmp[16];
    bal_to_native(cameras + 9 * i, tmp);
    std::memcpy(&nat[(size_t)i * 15], tmp, 15 * sizeof(double));
  }
  timer.mark("native cameras");
  // light plan: decide on the device whether the input point numbering follows the cameras; if not, fall back
  // to the full host plan with the locality renumbering.  d_opt (the observations' points on the device)
  // becomes the camera side's point index.
  if (C->plan.point_side_deferred) {
    // the record staging buffer (64 B per observation) is allocated now and lends its memory to the setup
    // temporaries (no allocate / free churn at create)
    IterParams& Q = C->P;
    if (!pre) {
      Q.n_records = std::max<int64_t>(K, 1);
      if ((rc = dalloc(C, &Q.staging, 8 * (size_t)Q.n_records)) || (rc = dalloc(C, &d_opt, (size_t)Q.n_records)))
        return g_bail_line = __LINE__, bail(rc);
      if (h2d(C, d_opt, obs_pt, sizeof(int32_t) * (size_t)K) != cudaSuccess ||
          h2d(C, reinterpret_cast<int32_t*>(Q.staging), obs_cam, sizeof(int32_t) * (size_t)K) != cudaSuccess)
        return g_bail_line = __LINE__, bail(DABA_E_CUDA);
    }
    int32_t* d_ocam = reinterpret_cast<int32_t*>(Q.staging);
    // scratch after the K camera ids: N int32 keys + a counter; with more points than the buffer holds (isolated
    // points) or no observations the check is skipped (nothing to gather, the numbering is kept)
    const bool fits = K > 0 && sizeof(int32_t) * ((size_t)K + 8 + (size_t)N) + 64 <= 64 * (size_t)Q.n_records;
    const int64_t jumps = fits ? count_point_jumps_device(d_ocam, d_opt, K, (int32_t)N, point_far,
                                                          Q.staging + ((size_t)K + 7) / 2, C->stream)
                               : 0;
    if (jumps < 0) return g_bail_line = __LINE__, bail(DABA_E_CUDA);
    if (point_order != 0 && jumps * 4 >= N && N > 1) {  // scattered numbering: full plan, renumbered
      std::string e2 = plan_shard(M, N, K, obs_cam, obs_pt, cam_owner, pt_owner, rank, nranks, &C->plan, false);
      if (!e2.empty()) return g_bail_line = __LINE__, bail(DABA_E_INVALID_ARG);
      order_owned_points(&C->plan, obs_cam, true);
      Q.staging = nullptr;  // (re-allocated at its final size by the full path; this one stays until destroy)
    }
    timer.mark("device point-order check");
  }
  const ShardPlan& S = C->plan;
  IterParams& P = C->P;
  P.n_cams = (int32_t)S.cam_g.size();
  P.n_own_cams = S.n_own_cams;
  P.n_pts = (int32_t)S.pt_g.size();
  P.n_own_pts = S.n_own_pts;
  P.loss = loss.kind;
  P.delta = loss.scale;
  P.delta2 = loss.scale * loss.scale;
  P.idelta2 = 1.0 / P.delta2;
  P.xi = o.xi;
  P.eta = o.eta;
  P.mu0 = o.lm_mu0;
  P.mu_up = o.lm_mu_up;
  P.eps2 = o.eps * o.eps;
  P.max_trials = o.lm_max_trials;
  P.accelerate = o.accelerate ? 1 : 0;
  P.restart_scope = o.restart_scope;
  for (int r = 0; r < 4; ++r) {
    if ((rc = dalloc(C, &P.cams[r], (size_t)P.n_cams * kCamStride))) return g_bail_line = __LINE__, bail(rc);
    if ((rc = dalloc(C, &P.pts[r], (size_t)P.n_pts))) return g_bail_line = __LINE__, bail(rc);
  }
  for (int r = 0; r < 3; ++r)
    if ((rc = dalloc(C, &P.cbarb[r], (size_t)P.n_cams * kCamStride))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.counter, 1))) return g_bail_line = __LINE__, bail(rc);
  cudaMemsetAsync(P.counter, 0, sizeof(int32_t), C->stream);
  P.has_comm = C->comm ? 1 : 0;
  for (int r = 0; r < 3; ++r)
    if ((rc = dalloc(C, &P.lbar[r], (size_t)P.n_pts))) return g_bail_line = __LINE__, bail(rc);
  {
    std::vector<int32_t> roles = {0, 1, 2, 3, 0, 1, 2};
    if ((rc = upload(C, &P.roles, roles))) return g_bail_line = __LINE__, bail(rc);
  }
  timer.mark("device, stream, comm");
  bool uv_on_side = false;  // the pixels' upload runs on the side stream (joined before the first objective)
  // camera side + chunks
  const int64_t chunk_obs = std::max<int64_t>(64, std::min<int64_t>(kCamChunkObs, env_int("DABA_CHUNK_OBS", kCamChunkObs)));
  {
    const bool light = S.point_side_deferred;
    const size_t kc = light ? (size_t)K : S.c_obs.size();
    double2* duv;
    int32_t* dpt = d_opt;
    if ((rc = dalloc(C, &duv, kc))) return g_bail_line = __LINE__, bail(rc);
    if (!light) {
      if ((rc = dalloc(C, &dpt, kc))) return g_bail_line = __LINE__, bail(rc);
      CUDA_OR(C, h2d(C, dpt, S.c_pt.data(), kc * sizeof(int32_t)));
    }
    if (S.cam_side_identity) {
      // one rank, input sorted by (camera, point): the camera-side pixels are the input itself (no host copy).
      // From page-locked memory the copy runs on the side stream, beside the device sort of the point side; the
      // main stream waits for it before the first objective evaluation.
      if (kc * sizeof(double2) >= (8u << 20) && is_pinned(obs_uv)) {
        CUDA_OR(C, cudaEventRecord(C->ev_fork0, C->stream));  // (after duv's stream-ordered allocation)
        CUDA_OR(C, cudaStreamWaitEvent(C->side, C->ev_fork0, 0) == cudaSuccess
                       ? cudaMemcpyAsync(duv, obs_uv, kc * sizeof(double2), cudaMemcpyHostToDevice, C->side)
                       : cudaErrorUnknown);
        CUDA_OR(C, cudaEventRecord(C->ev_join0, C->side));
        uv_on_side = true;
      } else {
        CUDA_OR(C, h2d(C, duv, obs_uv, kc * sizeof(double2)));
      }
    } else {
      hvec<double2> uv(kc);
      parallel_for((int64_t)kc, [&](int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q) uv[q] = make_double2(obs_uv[2 * S.c_obs[q]], obs_uv[2 * S.c_obs[q] + 1]);
      });
      CUDA_OR(C, h2d(C, duv, uv.data(), kc * sizeof(double2)));
      CUDA_OR(C, cudaStreamSynchronize(C->stream));  // uv is freed at the end of this scope
    }
    P.c_uv = duv;
    P.c_pt = dpt;
    std::vector<CamChunk> chunks;
    std::vector<int32_t> cptr(1, 0);
    for (int32_t i = 0; i < S.n_own_cams; ++i) {
      // balanced chunks: a camera's observations split into equal parts of at most chunk_obs (<= kCamChunkObs)
      const int64_t b = S.cam_ptr[(size_t)i], e = S.cam_ptr[(size_t)i + 1];
      const int64_t parts = (e - b + chunk_obs - 1) / chunk_obs;
      for (int64_t q = 0; q < parts; ++q) {
        CamChunk ch;
        ch.cam = i;
        ch.o0 = b + (e - b) * q / parts;
        ch.n = (int32_t)(b + (e - b) * (q + 1) / parts - ch.o0);
        chunks.push_back(ch);
      }
      cptr.push_back((int32_t)chunks.size());
    }
    P.n_chunks = (int32_t)chunks.size();
    // one CTA per chunk for both anchors once the chunks fill the GPU four times over (6 CTAs per SM)
    P.cam_shared_ctas = (int32_t)env_int("DABA_CAM_SHARED", P.n_chunks >= 4 * 6 * C->num_sms ? 1 : 0);
    const CamChunk* dch;
    if ((rc = upload(C, const_cast<CamChunk**>(&dch), chunks))) return g_bail_line = __LINE__, bail(rc);
    P.chunks = dch;
    const int32_t* dcp;
    if ((rc = upload(C, const_cast<int32_t**>(&dcp), cptr))) return g_bail_line = __LINE__, bail(rc);
    P.cam_chunk_ptr = dcp;
  }
  timer.mark("camera side");
  // point side: records written by the camera pass at its observation index; boundary observations (camera
  // owned elsewhere) are recomputed into records n_cam_side + b
  std::vector<int32_t> bcam, bpt;
  std::vector<double2> buv;
  {
    if (S.point_side_deferred) {  // light plan: every point's records in camera order, sorted on the device
      int64_t* dptr;
      int32_t* dsrc;
      if ((rc = dalloc(C, &dptr, (size_t)N + 1)) || (rc = dalloc(C, &dsrc, (size_t)std::max<int64_t>(K, 1))))
        return g_bail_line = __LINE__, bail(rc);
      if (sort_point_side_device(d_opt, K, (int32_t)N, dsrc, dptr, P.staging, 64 * (size_t)P.n_records,
                                 C->stream) != 0)
        return g_bail_line = __LINE__, bail(DABA_E_CUDA);
      P.p_ptr = dptr;
      P.p_src = dsrc;
      P.n_cam_side = K;
      P.n_boundary = 0;
      const int32_t *d1, *d2;
      const double2* d4;
      if ((rc = upload(C, const_cast<int32_t**>(&d1), bcam)) || (rc = upload(C, const_cast<int32_t**>(&d2), bpt)) ||
          (rc = upload(C, const_cast<double2**>(&d4), buv)))
        return g_bail_line = __LINE__, bail(rc);
      P.b_cam = d1;
      P.b_pt = d2;
      P.b_uv = d4;
    } else {
    const size_t kp = S.p_obs.size(), kc = S.c_obs.size();
    const int64_t* dptr;
    if ((rc = upload(C, const_cast<int64_t**>(&dptr), S.pt_ptr))) return g_bail_line = __LINE__, bail(rc);
    P.p_ptr = dptr;
    hvec<int32_t> src(kp);
    if (S.cam_side_identity) {  // the camera-side index of observation o is o
      parallel_for((int64_t)kp, [&](int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q) src[q] = S.p_obs[q];
      });
    } else {
      hvec<int32_t> cam_side_of((size_t)K);
      parallel_for(K, [&](int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q) cam_side_of[(size_t)q] = -1;
      });
      parallel_for((int64_t)kc, [&](int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q) cam_side_of[(size_t)S.c_obs[q]] = (int32_t)q;
      });
      parallel_for((int64_t)kp, [&](int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q) src[q] = cam_side_of[(size_t)S.p_obs[q]];
      });
    }
    for (size_t q = 0; q < (S.cam_side_identity ? 0 : kp); ++q) {
      if (src[q] >= 0) continue;  // written by this rank's camera pass
      src[q] = (int32_t)(kc + bcam.size());
      bcam.push_back(S.p_cam[q]);
      bpt.push_back(S.p_pt[q]);
      buv.push_back(make_double2(obs_uv[2 * S.p_obs[q]], obs_uv[2 * S.p_obs[q] + 1]));
    }
    if (bcam.size() > 1 && env_int("DABA_BSORT", 1) != 0) {
      // boundary observations in camera order (stable): neighbouring threads of k_pt_boundary then share the halo
      // camera's record in L1; the point side's record indices follow the permutation
      std::vector<int32_t> perm(bcam.size()), rank_of(bcam.size());
      for (size_t b = 0; b < perm.size(); ++b) perm[b] = (int32_t)b;
      std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return bcam[(size_t)x] < bcam[(size_t)y]; });
      std::vector<int32_t> c2(bcam.size()), p2(bcam.size());
      std::vector<double2> u2(bcam.size());
      for (size_t r = 0; r < perm.size(); ++r) {
        rank_of[(size_t)perm[r]] = (int32_t)r;
        c2[r] = bcam[(size_t)perm[r]];
        p2[r] = bpt[(size_t)perm[r]];
        u2[r] = buv[(size_t)perm[r]];
      }
      bcam.swap(c2);
      bpt.swap(p2);
      buv.swap(u2);
      for (size_t q = 0; q < src.size(); ++q)
        if (src[q] >= (int32_t)kc) src[q] = (int32_t)kc + rank_of[(size_t)(src[q] - (int32_t)kc)];
    }
    P.n_cam_side = (int64_t)kc;
    P.n_boundary = (int64_t)bcam.size();
    P.n_records = std::max<int64_t>(P.n_cam_side + P.n_boundary, 1);
    if ((rc = dalloc(C, &P.staging, 8 * (size_t)P.n_records))) return g_bail_line = __LINE__, bail(rc);
    const int32_t *d0, *d1, *d2;
    const double2* d4;
    if ((rc = upload(C, const_cast<int32_t**>(&d0), src)) || (rc = upload(C, const_cast<int32_t**>(&d1), bcam)) ||
        (rc = upload(C, const_cast<int32_t**>(&d2), bpt)) || (rc = upload(C, const_cast<double2**>(&d4), buv)))
      return g_bail_line = __LINE__, bail(rc);
    P.p_src = d0;
    P.b_cam = d1;
    P.b_pt = d2;
    P.b_uv = d4;
    }
    const size_t kc = S.point_side_deferred ? (size_t)K : S.c_obs.size();  // camera-side observations
    // per-device restart: the inter-device pairs of this rank (camera side with a halo point: sign +1; point
    // side with a halo camera: sign -1)
    if (P.restart_scope == 1) {
      std::vector<int32_t> ic, ip, is;
      std::vector<double2> iu;
      for (size_t q = 0; q < (S.point_side_deferred ? 0 : kc); ++q)  // (a light plan has no halo)
        if (S.c_pt[q] >= S.n_own_pts) {
          ic.push_back(S.c_cam[q]);
          ip.push_back(S.c_pt[q]);
          iu.push_back(make_double2(obs_uv[2 * S.c_obs[q]], obs_uv[2 * S.c_obs[q] + 1]));
          is.push_back(1);
        }
      for (size_t b = 0; b < bcam.size(); ++b) {
        ic.push_back(bcam[b]);
        ip.push_back(bpt[b]);
        iu.push_back(buv[b]);
        is.push_back(-1);
      }
      P.n_inter = (int64_t)ic.size();
      P.n_inter_blocks = (int32_t)((P.n_inter + kInterThreads - 1) / kInterThreads);
      const int32_t *e0, *e1, *e2;
      const double2* e3;
      if ((rc = upload(C, const_cast<int32_t**>(&e0), ic)) || (rc = upload(C, const_cast<int32_t**>(&e1), ip)) ||
          (rc = upload(C, const_cast<int32_t**>(&e2), is)) || (rc = upload(C, const_cast<double2**>(&e3), iu)) ||
          (rc = dalloc(C, &P.inter_part, 2 * (size_t)std::max(P.n_inter_blocks, 1))))
        return g_bail_line = __LINE__, bail(rc);
      P.i_cam = e0;
      P.i_pt = e1;
      P.i_sign = e2;
      P.i_uv = e3;
    }
    // point-pass grid: every thread a few points (grid-stride), at least 8 CTAs per SM's worth; measured on
    // Final-13682: 4.46M points 1184 -> 4352 CTAs -17 us, 0.58M points (8 ranks) 1184 better than 2264
    const int32_t pt_cap = (int32_t)env_int(
        "DABA_PT_CAP", std::max<int64_t>(148 * 8, ((int64_t)P.n_own_pts + 4 * kPtPassThreads - 1) / (4 * kPtPassThreads)));
    P.n_pt_blocks = std::max(1, std::min((P.n_own_pts + kPtPassThreads - 1) / kPtPassThreads, pt_cap));
  }
  timer.mark("point side");
  // scratch
  P.n_cam_eval_blocks = (2 * P.n_own_cams + 127) / 128;  // k_cam_solve blocks
  P.trace_cap = 1024;
  if ((rc = dalloc(C, &P.partial, (size_t)std::max(P.n_chunks, 1) * 2 * kPartialStride))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.moments, (size_t)std::max(P.n_own_cams, 1) * 2 * kPartialStride))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.dP_mm, (size_t)std::max(P.n_own_cams, 1)))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.decisions, (size_t)std::max(P.n_own_cams, 1) * 2))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.cam_part, (size_t)std::max(P.n_cam_eval_blocks, 1) * kCamEvalCols))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.pt_part, (size_t)std::max(P.n_pt_blocks, 1) * kPtCols))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.local, kGlobalCols))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.global, kGlobalCols))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.trace, (size_t)P.trace_cap * kTraceCols))) return g_bail_line = __LINE__, bail(rc);
  if ((rc = dalloc(C, &P.sched, 8))) return g_bail_line = __LINE__, bail(rc);
  if (!C->comm) P.global = P.local;
  cudaMemsetAsync(P.decisions, 0xff, sizeof(int32_t) * 2 * std::max(P.n_own_cams, 1), C->stream);
  timer.mark("scratch");
  // halo plan: per peer a segment [cameras x 15 | points x 3] of the send / receive buffers; the pack and unpack
  // items of all peers are flattened so that one kernel does each
  if (nranks > 1) {
    std::vector<int32_t> sc, sp, rcm, rpt;
    std::vector<int64_t> sco, spo, rco, rpo;
    int64_t soff = 0, roff = 0;
    for (const Peer& pe : S.peers) {
      PeerSeg sg;
      sg.rank = pe.rank;
      sg.send_off = soff;
      sg.send_cnt = kHaloCam * (int64_t)pe.send_cams.size() + 6 * (int64_t)pe.send_pts.size();  // both candidates
      sg.recv_off = roff;
      sg.recv_cnt = kHaloCam * (int64_t)pe.recv_cams.size() + 6 * (int64_t)pe.recv_pts.size();
      for (size_t q = 0; q < pe.send_cams.size(); ++q) {
        sc.push_back(pe.send_cams[q]);
        sco.push_back(soff + kHaloCam * (int64_t)q);
      }
      for (size_t q = 0; q < pe.send_pts.size(); ++q) {
        sp.push_back(pe.send_pts[q]);
        spo.push_back(soff + kHaloCam * (int64_t)pe.send_cams.size() + 6 * (int64_t)q);
      }
      for (size_t q = 0; q < pe.recv_cams.size(); ++q) {
        rcm.push_back(pe.recv_cams[q]);
        rco.push_back(roff + kHaloCam * (int64_t)q);
      }
      for (size_t q = 0; q < pe.recv_pts.size(); ++q) {
        rpt.push_back(pe.recv_pts[q]);
        rpo.push_back(roff + kHaloCam * (int64_t)pe.recv_cams.size() + 6 * (int64_t)q);
      }
      soff += sg.send_cnt;
      roff += sg.recv_cnt;
      C->segs.push_back(sg);
    }
    C->n_send_cam = (int32_t)sc.size();
    C->n_send_pt = (int32_t)sp.size();
    C->n_recv_cam = (int32_t)rcm.size();
    C->n_recv_pt = (int32_t)rpt.size();
    if ((rc = upload(C, &C->d_send_cam, sc)) || (rc = upload(C, &C->d_send_pt, sp)) ||
        (rc = upload(C, &C->d_recv_cam, rcm)) || (rc = upload(C, &C->d_recv_pt, rpt)) ||
        (rc = upload(C, &C->d_send_cam_off, sco)) || (rc = upload(C, &C->d_send_pt_off, spo)) ||
        (rc = upload(C, &C->d_recv_cam_off, rco)) || (rc = upload(C, &C->d_recv_pt_off, rpo)))
      return g_bail_line = __LINE__, bail(rc);
    if ((rc = dalloc(C, &C->d_sendbuf, (size_t)std::max<int64_t>(soff, 1))) ||
        (rc = dalloc(C, &C->d_recvbuf, (size_t)std::max<int64_t>(roff, 1))))
      return g_bail_line = __LINE__, bail(rc);
    // global test: the solves write both candidates into the send slots themselves (no k_pack); per owned
    // variable the list of its slots
    if (P.restart_scope == 0 && !C->segs.empty()) {
      auto csr = [](int32_t n, const std::vector<int32_t>& idx, const std::vector<int64_t>& off,
                    std::vector<int32_t>& ptr, std::vector<int64_t>& o) {
        ptr.assign((size_t)n + 1, 0);
        for (int32_t v : idx) ++ptr[(size_t)v + 1];
        for (int32_t v = 0; v < n; ++v) ptr[(size_t)v + 1] += ptr[(size_t)v];
        o.resize(idx.size());
        std::vector<int32_t> pos(ptr.begin(), ptr.end() - 1);
        for (size_t q = 0; q < idx.size(); ++q) o[(size_t)pos[(size_t)idx[q]]++] = off[q];
      };
      std::vector<int32_t> cptr_s, pptr_s;
      std::vector<int64_t> coff_s, poff_s;
      csr(P.n_own_cams, sc, sco, cptr_s, coff_s);
      csr(P.n_own_pts, sp, spo, pptr_s, poff_s);
      const int32_t *a0, *a2;
      const int64_t *a1, *a3;
      if ((rc = upload(C, const_cast<int32_t**>(&a0), cptr_s)) || (rc = upload(C, const_cast<int64_t**>(&a1), coff_s)) ||
          (rc = upload(C, const_cast<int32_t**>(&a2), pptr_s)) || (rc = upload(C, const_cast<int64_t**>(&a3), poff_s)))
        return g_bail_line = __LINE__, bail(rc);
      P.cam_send_ptr = a0;
      P.cam_send_off = a1;
      P.pt_send_ptr = a2;
      P.pt_send_off = a3;
      P.sendbuf = C->d_sendbuf;
    }
  }
  timer.mark("halo plan");
  // state: x^{-1} = x^0 (Alg. 1)
  {
    rc = upload_states(C, nat.data(), points, nat.data(), points, 1, 0);
    if (rc) return g_bail_line = __LINE__, bail(rc);
  }
  timer.mark("states");
  // s^{(0)} = 1, F-bar^{(-1)} = F(x^0) (eq. Fainit, global form), k = 0
  double F0 = 0, nd = 0;
  if (uv_on_side) CUDA_OR(C, cudaStreamWaitEvent(C->stream, C->ev_join0, 0));
  if ((rc = compute_objective(C, &F0, &nd))) return g_bail_line = __LINE__, bail(rc);
  if (nd > 0) return g_bail_line = __LINE__, bail(DABA_E_DEGENERATE);  // Assumption 2: ||l_j - t_i|| <= eps for some pair
  if (P.restart_scope == 1) {
    // eq. Fainit per device: F-bar^{a(-1)} = F^{a(-1)} = E^a(x^{a(0)} | x^{(0)}) = F_kappa(x^0): the rank's
    // camera-side F with its inter-device pairs at weight 1/2 (k_inter at x^{-1} = x^0); D^{a(-1)} = 0
    launch_inter(P, C->stream);
    launch_reduce_inter(P, C->stream);
    double loc[kGlobalCols];
    if (cudaMemcpyAsync(loc, P.local, sizeof loc, cudaMemcpyDeviceToHost, C->stream) != cudaSuccess ||
        cudaStreamSynchronize(C->stream) != cudaSuccess)
      return g_bail_line = __LINE__, bail(DABA_E_CUDA);
    F0 = loc[0] + loc[10];
  }
  {
    const double sched[8] = {1.0, F0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (cudaMemcpyAsync(P.sched, sched, sizeof sched, cudaMemcpyHostToDevice, C->stream) != cudaSuccess)
      return g_bail_line = __LINE__, bail(DABA_E_CUDA);
    launch_lbar_all(P, C->stream);  // x-bar^0 = x^0 (gamma^{(0)} = 0)
    if (cudaStreamSynchronize(C->stream) != cudaSuccess) return g_bail_line = __LINE__, bail(DABA_E_CUDA);
  }
  timer.mark("objective, x-bar");
  // launches per iteration (for bookkeeping)
  {
    const bool unpack = C->n_recv_cam + C->n_recv_pt > 0, dev = P.restart_scope == 1;
    C->launches_per_iter = 3 - (P.n_chunks == 0) - (P.n_own_cams == 0) + (P.n_boundary > 0) +
                           (P.n_inter_blocks > 0) + (C->comm && (dev || !unpack) ? 1 : 0) +
                           (C->n_send_cam + C->n_send_pt > 0 && !P.sendbuf) + unpack;
  }
  *out = c.release();
  return DABA_OK;
}

static int iterate_impl(daba_ctx* c, int n, double* trace_rows) {
  if (!c) return DABA_E_INVALID_ARG;
  if (n < 0) return fail(c, DABA_E_INVALID_ARG, "n_iters < 0");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, DABA_E_CUDA, "cudaSetDevice");
  const bool graphable =
      c->opt.use_graph && !c->opt.profile && !c->graph_failed && (!c->comm || c->comm->capturable());
  int done = 0;
  while (done < n) {
    const int batch = std::min(n - done, c->P.trace_cap);
    if (graphable && !c->graph) {
      cudaGraph_t g = nullptr;
      CUDA_OR(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      int launches = 0;
      const int rc = enqueue_iteration(c, &launches);
      cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
      if (rc == DABA_OK && ce == cudaSuccess) ce = cudaGraphInstantiate(&c->graph, g, 0);
      if (g) cudaGraphDestroy(g);
      if (rc != DABA_OK || ce != cudaSuccess || !c->graph) {
        // Capture is an optimisation: on failure (e.g. a transport that cannot be captured) launch the same
        // kernels eagerly from now on.  Nothing was executed during the failed capture.
        cudaGetLastError();
        c->graph = nullptr;
        c->graph_failed = true;
        fprintf(stderr, "daba: iteration graph capture failed (%s); launching eagerly\n",
                rc != DABA_OK ? c->err.c_str() : cudaGetErrorString(ce));
      }
    }
    if (c->graph) {
      for (int it = 0; it < batch; ++it) CUDA_OR(c, cudaGraphLaunch(c->graph, c->stream));
    } else {
      for (int it = 0; it < batch; ++it) {
        int launches = 0;
        int rc = enqueue_iteration(c, &launches);
        if (rc) return rc;
      }
    }
    if (trace_rows) {
      std::vector<double> ring((size_t)c->P.trace_cap * kTraceCols);
      CUDA_OR(c, cudaMemcpyAsync(ring.data(), c->P.trace, ring.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
      CUDA_OR(c, cudaStreamSynchronize(c->stream));
      for (int it = 0; it < batch; ++it) {
        const int64_t k = c->host_k + it;
        std::memcpy(trace_rows + (size_t)(done + it) * kTraceCols, &ring[(size_t)(k % c->P.trace_cap) * kTraceCols],
                    kTraceCols * sizeof(double));
      }
    }
    c->host_k += batch;
    done += batch;
  }
  if (c->opt.profile) collect_times(c);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return fail(c, DABA_E_CUDA, cudaGetErrorString(e));
  return DABA_OK;
}

extern "C" int daba_iterate(daba_ctx* ctx, int n_iters, double* F_trace, uint8_t* restart_trace) {
  if (!ctx) return DABA_E_INVALID_ARG;
  if (!F_trace && !restart_trace) return iterate_impl(ctx, n_iters, nullptr);
  std::vector<double> rows((size_t)std::max(n_iters, 0) * kTraceCols);
  int rc = iterate_impl(ctx, n_iters, rows.data());
  if (rc) return rc;
  for (int k = 0; k < n_iters; ++k) {
    if (F_trace) F_trace[k] = rows[(size_t)k * kTraceCols + DABA_TR_F];
    if (restart_trace) restart_trace[k] = rows[(size_t)k * kTraceCols + DABA_TR_RESTART] != 0.0;
  }
  return DABA_OK;
}

extern "C" int daba_iterate_trace(daba_ctx* ctx, int n_iters, double* trace) {
  if (!ctx || !trace) return DABA_E_INVALID_ARG;
  return iterate_impl(ctx, n_iters, trace);
}

extern "C" int daba_objective(daba_ctx* ctx, double* F_out) {
  if (!ctx || !F_out) return DABA_E_INVALID_ARG;
  cudaSetDevice(ctx->device);
  return compute_objective(ctx, F_out, nullptr);
}

extern "C" int daba_pixel_error(daba_ctx* ctx, double out[4]) {
  if (!ctx || !out) return DABA_E_INVALID_ARG;
  cudaSetDevice(ctx->device);
  int rc;
  if (!ctx->d_metric && (rc = dalloc(ctx, &ctx->d_metric, 4))) return rc;
  launch_pixel_error(ctx->P, 1, ctx->d_metric, nullptr, ctx->stream);
  CUDA_OR(ctx, cudaGetLastError());
  CUDA_OR(ctx, cudaMemcpyAsync(out, ctx->d_metric, 4 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OR(ctx, cudaStreamSynchronize(ctx->stream));
  return DABA_OK;
}

extern "C" int daba_pixel_residuals(daba_ctx* ctx, double* resid_out) {
  if (!ctx || !resid_out) return DABA_E_INVALID_ARG;
  cudaSetDevice(ctx->device);
  const ShardPlan& S = ctx->plan;
  const bool identity = S.point_side_deferred || S.cam_side_identity;
  const int64_t kc = ctx->P.n_cam_side;
  if (kc == 0) return DABA_OK;
  if (!ctx->P.staging || (size_t)kc > 8 * (size_t)ctx->P.n_records) return fail(ctx, DABA_E_STATE, "no scratch");
  int rc;
  if (!ctx->d_metric && (rc = dalloc(ctx, &ctx->d_metric, 4))) return rc;
  // per-observation residuals in the record staging buffer (free between iterations)
  launch_pixel_error(ctx->P, 1, ctx->d_metric, ctx->P.staging, ctx->stream);
  CUDA_OR(ctx, cudaGetLastError());
  if (identity) {
    CUDA_OR(ctx, d2h(ctx, resid_out, ctx->P.staging, (size_t)kc * sizeof(double)));
    return DABA_OK;
  }
  hvec<double> h((size_t)kc);
  CUDA_OR(ctx, d2h(ctx, h.data(), ctx->P.staging, (size_t)kc * sizeof(double)));
  parallel_for(kc, [&](int64_t a, int64_t b) {
    for (int64_t q = a; q < b; ++q) resid_out[S.c_obs[(size_t)q]] = h[(size_t)q];
  });
  return DABA_OK;
}

// Reads the owned cameras (native records) into hc and, unless the points go straight to the caller, the owned
// points into hp.  With the light plan (one rank, identity numbering) the points are packed to xyz on the device
// (in the record staging buffer, free between iterations) and copied once into points_out: *direct = true.
static int get_native(daba_ctx* c, int which, hvec<double>& hc, hvec<double>& hp, double* points_out, bool* direct) {
  int roles[4];
  CUDA_OR(c, cudaMemcpyAsync(roles, c->P.roles, sizeof roles, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR(c, cudaStreamSynchronize(c->stream));
  const int r = roles[which ? 0 : 1];
  const ShardPlan& S = c->plan;
  const int32_t np = c->P.n_own_pts;
  *direct = S.point_side_deferred && np == S.N && c->P.staging &&
            3 * (size_t)np <= 8 * (size_t)c->P.n_records;
  hc.resize((size_t)c->P.n_own_cams * kCamStride);
  if (!hc.empty())
    CUDA_OR(c, cudaMemcpyAsync(hc.data(), c->P.cams[r], hc.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (*direct) {
    if (points_out && np > 0) {
      launch_pts_xyz(c->P.pts[r], c->P.staging, np, c->stream);
      CUDA_OR(c, cudaGetLastError());
      CUDA_OR(c, d2h(c, points_out, c->P.staging, 3 * (size_t)np * sizeof(double)));
    }
  } else {
    hp.resize((size_t)np * 4);
    if (!hp.empty()) CUDA_OR(c, d2h(c, hp.data(), c->P.pts[r], hp.size() * sizeof(double)));
  }
  CUDA_OR(c, cudaStreamSynchronize(c->stream));
  return DABA_OK;
}

// points of the host copy (not direct) to their global slots, and the owned mask
static void scatter_points(const ShardPlan& S, const hvec<double>& hp, bool direct, double* points_out,
                           uint8_t* owned_mask_out) {
  if (direct) {
    if (owned_mask_out) std::memset(owned_mask_out + S.M, 1, (size_t)S.N);
    return;
  }
  parallel_for(S.n_own_pts, [&](int64_t a, int64_t b) {
    for (int64_t lj = a; lj < b; ++lj) {
      const int64_t g = S.pt_g[(size_t)lj];
      if (points_out)
        for (int k = 0; k < 3; ++k) points_out[3 * g + k] = hp[(size_t)lj * 4 + k];
      if (owned_mask_out) owned_mask_out[S.M + g] = 1;
    }
  });
}

extern "C" int daba_get_state_native(daba_ctx* ctx, int which, double* cameras_out, double* points_out,
                                     uint8_t* owned_mask_out) {
  if (!ctx || which < 0 || which > 1) return DABA_E_INVALID_ARG;
  cudaSetDevice(ctx->device);
  hvec<double> hc, hp;
  bool direct = false;
  int rc = get_native(ctx, which, hc, hp, points_out, &direct);
  if (rc) return rc;
  const ShardPlan& S = ctx->plan;
  if (owned_mask_out) std::memset(owned_mask_out, 0, (size_t)(S.M + S.N));
  for (int32_t li = 0; li < S.n_own_cams; ++li) {
    const int64_t g = S.cam_g[(size_t)li];
    if (cameras_out) std::memcpy(cameras_out + 15 * g, &hc[(size_t)li * kCamStride], 15 * sizeof(double));
    if (owned_mask_out) owned_mask_out[g] = 1;
  }
  scatter_points(S, hp, direct, points_out, owned_mask_out);
  return DABA_OK;
}

extern "C" int daba_get_state(daba_ctx* ctx, double* cameras_out, double* points_out, uint8_t* owned_mask_out) {
  if (!ctx) return DABA_E_INVALID_ARG;
  cudaSetDevice(ctx->device);
  hvec<double> hc, hp;
  bool direct = false;
  int rc = get_native(ctx, 0, hc, hp, points_out, &direct);
  if (rc) return rc;
  const ShardPlan& S = ctx->plan;
  if (owned_mask_out) std::memset(owned_mask_out, 0, (size_t)(S.M + S.N));
  for (int32_t li = 0; li < S.n_own_cams; ++li) {
    const int64_t g = S.cam_g[(size_t)li];
    if (cameras_out) native_to_bal(&hc[(size_t)li * kCamStride], cameras_out + 9 * g);
    if (owned_mask_out) owned_mask_out[g] = 1;
  }
  scatter_points(S, hp, direct, points_out, owned_mask_out);
  return DABA_OK;
}

extern "C" int daba_set_state_native(daba_ctx* ctx, const double* cams_k, const double* pts_k,
                                     const double* cams_km1, const double* pts_km1, double s, double Fbar) {
  if (!ctx || (ctx->plan.M > 0 && (!cams_k || !cams_km1)) || (ctx->plan.N > 0 && (!pts_k || !pts_km1)) || !(s >= 1))
    return DABA_E_INVALID_ARG;
  if (ctx->P.restart_scope == 1)
    return fail(ctx, DABA_E_STATE, "daba_set_state_native: the per-device restart metrics cannot be restored");
  cudaSetDevice(ctx->device);
  int rc = upload_states(ctx, cams_k, pts_k, cams_km1, pts_km1, 1, 0);
  if (rc) return rc;
  double sched[3];
  CUDA_OR(ctx, cudaMemcpyAsync(sched, ctx->P.sched, sizeof sched, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OR(ctx, cudaStreamSynchronize(ctx->stream));
  sched[0] = s;
  sched[1] = Fbar;
  CUDA_OR(ctx, cudaMemcpyAsync(ctx->P.sched, sched, sizeof sched, cudaMemcpyHostToDevice, ctx->stream));
  launch_lbar_all(ctx->P, ctx->stream);  // x-bar^k of the resumed state
  CUDA_OR(ctx, cudaStreamSynchronize(ctx->stream));
  return DABA_OK;
}

extern "C" int daba_get_schedule(daba_ctx* ctx, double* s, double* Fbar, int64_t* k) {
  if (!ctx) return DABA_E_INVALID_ARG;
  double sched[4];
  CUDA_OR(ctx, cudaMemcpyAsync(sched, ctx->P.sched, sizeof sched, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OR(ctx, cudaStreamSynchronize(ctx->stream));
  if (s) *s = sched[0];
  if (Fbar) *Fbar = sched[1];
  if (k) *k = (int64_t)sched[2];
  return DABA_OK;
}

extern "C" int daba_last_decisions(daba_ctx* ctx, int32_t* trial_acc, int32_t* trial_mm) {
  if (!ctx) return DABA_E_INVALID_ARG;
  std::vector<int32_t> d((size_t)std::max(ctx->P.n_own_cams, 1) * 2);
  CUDA_OR(ctx, cudaMemcpyAsync(d.data(), ctx->P.decisions, d.size() * sizeof(int32_t), cudaMemcpyDeviceToHost,
                               ctx->stream));
  CUDA_OR(ctx, cudaStreamSynchronize(ctx->stream));
  for (int32_t li = 0; li < ctx->P.n_own_cams; ++li) {
    const int64_t g = ctx->plan.cam_g[(size_t)li];
    if (trial_acc) trial_acc[g] = d[(size_t)2 * li];
    if (trial_mm) trial_mm[g] = d[(size_t)2 * li + 1];
  }
  return DABA_OK;
}

extern "C" int daba_shard_info(daba_ctx* ctx, int64_t info[8]) {
  if (!ctx || !info) return DABA_E_INVALID_ARG;
  const ShardPlan& S = ctx->plan;
  info[0] = S.n_own_cams;
  info[1] = S.n_own_pts;
  info[2] = (int64_t)S.cam_g.size() - S.n_own_cams;
  info[3] = (int64_t)S.pt_g.size() - S.n_own_pts;
  info[4] = S.point_side_deferred ? S.K : (int64_t)S.c_obs.size();
  info[5] = S.point_side_deferred ? S.K : (int64_t)S.p_obs.size();
  info[6] = 16 * S.send_doubles;  // both candidates of each boundary variable, 8 B each
  info[7] = (int64_t)ctx->dev_bytes;
  return DABA_OK;
}

extern "C" void* daba_stream(daba_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

extern "C" int daba_kernel_times(daba_ctx* ctx, char* names_out, size_t cap, double* ms_out, int64_t* launches_out) {
  if (!ctx) return DABA_E_INVALID_ARG;
  collect_times(ctx);
  std::string all;
  const int n = (int)std::min<size_t>(ctx->knames.size(), 32);
  for (int i = 0; i < n; ++i) {
    all += ctx->knames[(size_t)i];
    all += '\n';
    if (ms_out) ms_out[i] = ctx->kms[(size_t)i];
    if (launches_out) launches_out[i] = ctx->klaunches[(size_t)i];
  }
  if (names_out && cap > 0) {
    std::strncpy(names_out, all.c_str(), cap - 1);
    names_out[cap - 1] = 0;
  }
  return n;
}

extern "C" int daba_reset_kernel_times(daba_ctx* ctx) {
  if (!ctx) return DABA_E_INVALID_ARG;
  collect_times(ctx);
  std::fill(ctx->kms.begin(), ctx->kms.end(), 0.0);
  std::fill(ctx->klaunches.begin(), ctx->klaunches.end(), 0);
  return DABA_OK;
}

extern "C" int daba_launches_per_iteration(daba_ctx* ctx) { return ctx ? ctx->launches_per_iter : DABA_E_INVALID_ARG; }

extern "C" const char* daba_last_error(const daba_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

extern "C" void daba_destroy(daba_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->side) cudaStreamSynchronize(ctx->side);  // (a create that failed with a side-stream upload in flight)
  collect_times(ctx);
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
  ctx->comm.reset();
  if (ctx->pooled && ctx->stream) {
    for (void* p : ctx->allocs) cudaFreeAsync(p, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
  } else {
    for (void* p : ctx->allocs) cudaFree(p);
  }
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_fork0) cudaEventDestroy(ctx->ev_fork0);
  if (ctx->ev_join0) cudaEventDestroy(ctx->ev_join0);
  delete ctx;
}

// The same retained pool for the stateless NEXT-3 entry points (coarse.cu).
namespace daba {
cudaMemPool_t shared_pool(int device) { return context_pool(device); }
}  // namespace daba
