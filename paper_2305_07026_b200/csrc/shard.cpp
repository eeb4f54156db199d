// shard.cpp — host-side partition and halo plan (see shard.h).
//
// Linear-time passes over the observations (counting sorts); the common case of input already sorted by
// (camera, point) skips the camera sort.
#include "shard.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <thread>

namespace daba {

namespace {

// Split [0, n) over the host's cores (small n: one thread).
template <class F>
void pfor(int64_t n, F&& f, int64_t work = -1) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if ((work < 0 ? n : work) < (1 << 16) || hw == 1 || n < (int64_t)hw) {
    f(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (unsigned t = 0; t < hw; ++t) th.emplace_back([&, t] { f(n * t / hw, n * (t + 1) / hw, (int)t); });
  for (auto& x : th) x.join();
}
unsigned nthreads(int64_t n) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  return (n < (1 << 16) || hw == 1) ? 1u : hw;
}

// Stable sort of observation ids by key (0..nkeys-1); ptr gets nkeys+1 offsets.  Parallel LSD radix sort on
// (key, id) pairs, <= 13 bits per pass (two passes up to 2^26 keys): per-thread digit histograms over contiguous input slices, then a stable
// scatter (thread t writes its slice's elements in order after threads < t) — sequential streams, no atomics.
void bucket(int64_t nkeys, const hvec<int32_t>& ids, const int32_t* key, std::vector<int64_t>& ptr,
            hvec<int32_t>& out) {
  const int64_t n = (int64_t)ids.size();
  hvec<int32_t> k0((size_t)n), v0((size_t)n), k1((size_t)n), v1((size_t)n);
  pfor(n, [&](int64_t a, int64_t b, int) {
    for (int64_t q = a; q < b; ++q) {
      v0[(size_t)q] = ids[(size_t)q];
      k0[(size_t)q] = key[ids[(size_t)q]];
    }
  });
  int bits = 1;
  while ((int64_t(1) << bits) < nkeys) ++bits;
  const int passes = (bits + 12) / 13;               // <= 13 bits per pass (8192 buckets per thread)
  const int R = (bits + passes - 1) / passes, B = 1 << R;
  const unsigned T = nthreads(n);
  std::vector<int64_t> hist((size_t)T * B);
  for (int shift = 0; shift < bits; shift += R) {
    std::fill(hist.begin(), hist.end(), 0);
    pfor(n, [&](int64_t a, int64_t b, int t) {
      int64_t* h = &hist[(size_t)t * B];
      for (int64_t q = a; q < b; ++q) ++h[(k0[(size_t)q] >> shift) & (B - 1)];
    });
    int64_t run = 0;  // digit-major, thread-minor exclusive prefix: stable
    for (int d = 0; d < B; ++d)
      for (unsigned t = 0; t < T; ++t) {
        const int64_t c = hist[(size_t)t * B + d];
        hist[(size_t)t * B + d] = run;
        run += c;
      }
    pfor(n, [&](int64_t a, int64_t b, int t) {
      int64_t* h = &hist[(size_t)t * B];
      for (int64_t q = a; q < b; ++q) {
        const int64_t w = h[(k0[(size_t)q] >> shift) & (B - 1)]++;
        k1[(size_t)w] = k0[(size_t)q];
        v1[(size_t)w] = v0[(size_t)q];
      }
    });
    k0.swap(k1);
    v0.swap(v1);
  }
  out.swap(v0);
  ptr.assign((size_t)nkeys + 1, 0);
  // offsets: the first position of every key present (keys ascending), then fill the gaps of absent keys
  pfor(n, [&](int64_t a, int64_t b, int) {
    for (int64_t q = a; q < b; ++q)
      if (q == 0 || k0[(size_t)q] != k0[(size_t)q - 1]) ptr[(size_t)k0[(size_t)q]] = q;
  });
  // keys without entries take the next key's start; walk backwards (serial, nkeys steps)
  int64_t next = n;
  std::vector<uint8_t> present((size_t)nkeys, 0);
  pfor(n, [&](int64_t a, int64_t b, int) {
    for (int64_t q = a; q < b; ++q)
      if (q == 0 || k0[(size_t)q] != k0[(size_t)q - 1]) present[(size_t)k0[(size_t)q]] = 1;
  });
  ptr[(size_t)nkeys] = n;
  for (int64_t k = nkeys - 1; k >= 0; --k) {
    if (!present[(size_t)k]) ptr[(size_t)k] = next;
    next = ptr[(size_t)k];
  }
}

struct Tm {
  bool on = std::getenv("DABA_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* w) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "plan_shard %-20s %8.1f ms\n", w, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

}  // namespace

void plan_light(int64_t M, int64_t N, int64_t K, std::vector<int64_t> cam_ptr, ShardPlan* out) {
  ShardPlan& P = *out;
  P = ShardPlan();
  P.M = M;
  P.N = N;
  P.K = K;
  P.cam_owner.assign((size_t)M, 0);
  P.pt_owner.assign((size_t)N, 0);
  P.cam_g.resize((size_t)M);
  P.pt_g.resize((size_t)N);
  pfor(M, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; ++i) P.cam_g[(size_t)i] = (int32_t)i;
  });
  pfor(N, [&](int64_t a, int64_t b, int) {
    for (int64_t j = a; j < b; ++j) P.pt_g[(size_t)j] = (int32_t)j;
  });
  P.n_own_cams = (int32_t)M;
  P.n_own_pts = (int32_t)N;
  P.cam_ptr = std::move(cam_ptr);
  P.cam_side_identity = true;
  P.point_side_deferred = true;
}

std::string plan_shard(int64_t M, int64_t N, int64_t K, const int32_t* obs_cam, const int32_t* obs_pt,
                       const int32_t* cam_owner_in, const int32_t* pt_owner_in, int rank, int nranks,
                       ShardPlan* out, bool defer_point_side) {
  char msg[256];
  Tm tm;
  if (M < 0 || N < 0 || K < 0 || nranks < 1 || rank < 0 || rank >= nranks) return "invalid sizes or rank";
  if (M > INT32_MAX - 1 || N > INT32_MAX - 1 || K > INT32_MAX - 1) return "M, N and K must be < 2^31 - 1";
  if (K > 0 && (!obs_cam || !obs_pt)) return "null observation arrays";
  ShardPlan& P = *out;
  P = ShardPlan();
  P.rank = rank;
  P.nranks = nranks;
  P.M = M;
  P.N = N;
  P.K = K;
  // ---- validation, and whether the input is already sorted by (camera, point), strictly
  std::atomic<int64_t> bad(K);
  std::atomic<bool> sorted(true);
  pfor(K, [&](int64_t a, int64_t b, int) {
    bool srt = true;
    for (int64_t k = a; k < b; ++k) {
      if (obs_cam[k] < 0 || obs_cam[k] >= M || obs_pt[k] < 0 || obs_pt[k] >= N) {
        int64_t cur = bad.load();
        while (k < cur && !bad.compare_exchange_weak(cur, k)) {
        }
        break;
      }
      if (k > 0 && srt && !(obs_cam[k - 1] < obs_cam[k] || (obs_cam[k - 1] == obs_cam[k] && obs_pt[k - 1] < obs_pt[k])))
        srt = false;
    }
    if (!srt) sorted = false;
  });
  if (bad.load() < K) {
    const int64_t k = bad.load();
    snprintf(msg, sizeof msg, "observation %lld has index out of range (camera %d, point %d)", (long long)k,
             obs_cam[k], obs_pt[k]);
    return msg;
  }
  tm.mark("validate");
  // ---- observations in (camera, point) order; duplicate (i,j) check
  const bool light = defer_point_side && sorted && nranks == 1 && !cam_owner_in && !pt_owner_in;
  hvec<int32_t> cam_sorted(light ? 0 : (size_t)K);
  std::vector<int64_t> cptr((size_t)M + 1, 0);
  if (sorted) {
    const unsigned T = nthreads(K);
    std::vector<std::vector<int64_t>> part(T, std::vector<int64_t>((size_t)M, 0));
    pfor(K, [&](int64_t a, int64_t b, int t) {
      std::vector<int64_t>& c = part[(size_t)t];
      for (int64_t k = a; k < b; ++k) {
        if (!light) cam_sorted[(size_t)k] = (int32_t)k;
        ++c[(size_t)obs_cam[k]];
      }
    });
    for (unsigned t = 0; t < T; ++t)
      for (int64_t i = 0; i < M; ++i) cptr[(size_t)i + 1] += part[t][(size_t)i];
    for (int64_t i = 0; i < M; ++i) cptr[(size_t)i + 1] += cptr[(size_t)i];
    if (light) {  // one rank owns everything in input order; the point side is the engine's (on the device)
      P.cam_owner.assign((size_t)M, 0);
      P.pt_owner.assign((size_t)N, 0);
      P.cam_g.resize((size_t)M);
      P.pt_g.resize((size_t)N);
      pfor(M, [&](int64_t a, int64_t b, int) {
        for (int64_t i = a; i < b; ++i) P.cam_g[(size_t)i] = (int32_t)i;
      });
      pfor(N, [&](int64_t a, int64_t b, int) {
        for (int64_t j = a; j < b; ++j) P.pt_g[(size_t)j] = (int32_t)j;
      });
      P.n_own_cams = (int32_t)M;
      P.n_own_pts = (int32_t)N;
      P.cam_ptr = cptr;
      P.cam_side_identity = true;
      P.point_side_deferred = true;
      tm.mark("light plan");
      return "";
    }
  } else {
    hvec<int32_t> all((size_t)K);
    pfor(K, [&](int64_t a, int64_t b, int) {
      for (int64_t k = a; k < b; ++k) all[(size_t)k] = (int32_t)k;
    });
    bucket(M, all, obs_cam, cptr, cam_sorted);
    std::atomic<int64_t> dup_cam(-1);
    pfor(M, [&](int64_t a, int64_t b, int) {
      for (int64_t i = a; i < b; ++i) {
        auto lo = cam_sorted.begin() + cptr[(size_t)i], hi = cam_sorted.begin() + cptr[(size_t)i + 1];
        std::stable_sort(lo, hi, [&](int32_t x, int32_t y) { return obs_pt[x] < obs_pt[y]; });
        for (auto it = lo; it + 1 < hi; ++it)
          if (obs_pt[*(it + 1)] == obs_pt[*it]) dup_cam = i;
      }
    });
    if (dup_cam.load() >= 0) {
      snprintf(msg, sizeof msg, "duplicate observation at camera %lld", (long long)dup_cam.load());
      return msg;
    }
  }
  tm.mark("camera order");
  // ---- camera ownership
  P.cam_owner.assign((size_t)M, 0);
  if (cam_owner_in) {
    for (int64_t i = 0; i < M; ++i) {
      if (cam_owner_in[i] < 0 || cam_owner_in[i] >= nranks) return "cam_owner entry out of range";
      P.cam_owner[(size_t)i] = cam_owner_in[i];
    }
  } else if (nranks > 1) {
    // contiguous ranges balanced by observation count: the midpoint of camera i's observation range
    // decides its rank; without observations, balance by camera count
    for (int64_t i = 0; i < M; ++i) {
      const double mid = K > 0 ? (double)cptr[(size_t)i] + 0.5 * (double)(cptr[(size_t)i + 1] - cptr[(size_t)i])
                               : (double)i + 0.5;
      const double tot = K > 0 ? (double)K : (double)M;
      int r = (int)(mid * nranks / tot);
      P.cam_owner[(size_t)i] = std::min(std::max(r, 0), nranks - 1);
    }
  }
  tm.mark("cam owner");
  // ---- point ownership (observations bucketed by point; stable, so cameras ascend within a point)
  hvec<int32_t> pt_sorted;
  std::vector<int64_t> pptr;
  bucket(N, cam_sorted, obs_pt, pptr, pt_sorted);
  P.pt_owner.assign((size_t)N, 0);
  if (pt_owner_in) {
    for (int64_t j = 0; j < N; ++j) {
      if (pt_owner_in[j] < 0 || pt_owner_in[j] >= nranks) return "pt_owner entry out of range";
      P.pt_owner[(size_t)j] = pt_owner_in[j];
    }
  } else if (nranks > 1) {
    pfor(N, [&](int64_t a, int64_t b, int) {
      std::vector<int64_t> cnt((size_t)nranks);
      for (int64_t j = a; j < b; ++j) {
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t q = pptr[(size_t)j]; q < pptr[(size_t)j + 1]; ++q)
          ++cnt[(size_t)P.cam_owner[(size_t)obs_cam[pt_sorted[(size_t)q]]]];
        int best = 0;
        for (int r = 1; r < nranks; ++r)
          if (cnt[(size_t)r] > cnt[(size_t)best]) best = r;  // ties -> lowest rank
        P.pt_owner[(size_t)j] = best;
      }
    });
  }
  tm.mark("point bucket+owner");
  // ---- local numbering: owned first (ascending global id), halo after
  std::vector<int32_t> g2l_cam((size_t)M, -1), g2l_pt((size_t)N, -1);
  for (int64_t i = 0; i < M; ++i)
    if (P.cam_owner[(size_t)i] == rank) {
      g2l_cam[(size_t)i] = (int32_t)P.cam_g.size();
      P.cam_g.push_back((int32_t)i);
    }
  {  // owned points in ascending id: per-thread counts, offsets, fills
    const unsigned T = nthreads(N);
    std::vector<int64_t> cnt((size_t)T + 1, 0);
    pfor(N, [&](int64_t a, int64_t b, int t) {
      int64_t c = 0;
      for (int64_t j = a; j < b; ++j) c += P.pt_owner[(size_t)j] == rank;
      cnt[(size_t)t + 1] = c;
    });
    for (unsigned t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
    P.pt_g.resize((size_t)cnt[T]);
    pfor(N, [&](int64_t a, int64_t b, int t) {
      int64_t w = cnt[(size_t)t];
      for (int64_t j = a; j < b; ++j)
        if (P.pt_owner[(size_t)j] == rank) {
          g2l_pt[(size_t)j] = (int32_t)w;
          P.pt_g[(size_t)w++] = (int32_t)j;
        }
    });
  }
  P.n_own_cams = (int32_t)P.cam_g.size();
  P.n_own_pts = (int32_t)P.pt_g.size();
  if (nranks > 1) {
    // halo points: read by the camera side; halo cameras: read by the point side (benign byte races)
    std::vector<uint8_t> need_pt((size_t)N, 0), need_cam((size_t)M, 0);
    pfor(K, [&](int64_t a, int64_t b, int) {
      for (int64_t q = a; q < b; ++q) {
        const int32_t i = obs_cam[q], j = obs_pt[q];
        const bool oc = P.cam_owner[(size_t)i] == rank, op = P.pt_owner[(size_t)j] == rank;
        if (oc && !op) need_pt[(size_t)j] = 1;
        if (op && !oc) need_cam[(size_t)i] = 1;
      }
    });
    for (int64_t j = 0; j < N; ++j)
      if (need_pt[(size_t)j]) {
        g2l_pt[(size_t)j] = (int32_t)P.pt_g.size();
        P.pt_g.push_back((int32_t)j);
      }
    for (int64_t i = 0; i < M; ++i)
      if (need_cam[(size_t)i]) {
        g2l_cam[(size_t)i] = (int32_t)P.cam_g.size();
        P.cam_g.push_back((int32_t)i);
      }
  }
  tm.mark("numbering+halo");
  // ---- camera side, point side (offsets first, then parallel fills)
  P.cam_ptr.assign((size_t)P.n_own_cams + 1, 0);
  for (int32_t li = 0; li < P.n_own_cams; ++li) {
    const int64_t gi = P.cam_g[(size_t)li];
    P.cam_ptr[(size_t)li + 1] = P.cam_ptr[(size_t)li] + (cptr[(size_t)gi + 1] - cptr[(size_t)gi]);
  }
  P.pt_ptr.assign((size_t)P.n_own_pts + 1, 0);
  for (int32_t lj = 0; lj < P.n_own_pts; ++lj) {
    const int64_t gj = P.pt_g[(size_t)lj];
    P.pt_ptr[(size_t)lj + 1] = P.pt_ptr[(size_t)lj] + (pptr[(size_t)gj + 1] - pptr[(size_t)gj]);
  }
  const int64_t kc = P.cam_ptr.back(), kp = P.pt_ptr.back();
  P.cam_side_identity = sorted && nranks == 1;
  P.c_cam.resize((size_t)kc);
  P.c_pt.resize((size_t)kc);
  P.c_obs.resize((size_t)kc);
  pfor(P.n_own_cams, [&](int64_t a, int64_t b, int) {
    for (int64_t li = a; li < b; ++li) {
      const int64_t gi = P.cam_g[(size_t)li];
      int64_t w = P.cam_ptr[(size_t)li];
      for (int64_t q = cptr[(size_t)gi]; q < cptr[(size_t)gi + 1]; ++q, ++w) {
        const int32_t o = cam_sorted[(size_t)q];
        P.c_cam[(size_t)w] = (int32_t)li;
        P.c_pt[(size_t)w] = g2l_pt[(size_t)obs_pt[o]];
        P.c_obs[(size_t)w] = o;
      }
    }
  }, kc);
  P.p_cam.resize((size_t)kp);
  P.p_pt.resize((size_t)kp);
  P.p_obs.resize((size_t)kp);
  pfor(P.n_own_pts, [&](int64_t a, int64_t b, int) {
    for (int64_t lj = a; lj < b; ++lj) {
      const int64_t gj = P.pt_g[(size_t)lj];
      int64_t w = P.pt_ptr[(size_t)lj];
      for (int64_t q = pptr[(size_t)gj]; q < pptr[(size_t)gj + 1]; ++q, ++w) {
        const int32_t o = pt_sorted[(size_t)q];
        P.p_cam[(size_t)w] = g2l_cam[(size_t)obs_cam[o]];
        P.p_pt[(size_t)w] = (int32_t)lj;
        P.p_obs[(size_t)w] = o;
      }
    }
  });
  tm.mark("sides");
  // ---- peers
  if (nranks > 1) {
    std::vector<std::vector<uint8_t>> sc((size_t)nranks, std::vector<uint8_t>((size_t)P.n_own_cams, 0));
    std::vector<std::vector<uint8_t>> sp((size_t)nranks, std::vector<uint8_t>((size_t)P.n_own_pts, 0));
    pfor((int64_t)P.c_obs.size(), [&](int64_t a, int64_t b, int) {
      for (int64_t q = a; q < b; ++q) {
        const int r = P.pt_owner[(size_t)obs_pt[P.c_obs[(size_t)q]]];
        if (r != rank) sc[(size_t)r][(size_t)P.c_cam[(size_t)q]] = 1;
      }
    });
    pfor((int64_t)P.p_obs.size(), [&](int64_t a, int64_t b, int) {
      for (int64_t q = a; q < b; ++q) {
        const int r = P.cam_owner[(size_t)obs_cam[P.p_obs[(size_t)q]]];
        if (r != rank) sp[(size_t)r][(size_t)P.p_pt[(size_t)q]] = 1;
      }
    });
    for (int b = 0; b < nranks; ++b) {
      if (b == rank) continue;
      Peer pe;
      pe.rank = b;
      for (int32_t li = 0; li < P.n_own_cams; ++li)
        if (sc[(size_t)b][(size_t)li]) pe.send_cams.push_back(li);
      for (int32_t lj = 0; lj < P.n_own_pts; ++lj)
        if (sp[(size_t)b][(size_t)lj]) pe.send_pts.push_back(lj);
      for (size_t li = (size_t)P.n_own_cams; li < P.cam_g.size(); ++li)
        if (P.cam_owner[(size_t)P.cam_g[li]] == b) pe.recv_cams.push_back((int32_t)li);
      for (size_t lj = (size_t)P.n_own_pts; lj < P.pt_g.size(); ++lj)
        if (P.pt_owner[(size_t)P.pt_g[lj]] == b) pe.recv_pts.push_back((int32_t)lj);
      if (pe.send_cams.empty() && pe.send_pts.empty() && pe.recv_cams.empty() && pe.recv_pts.empty()) continue;
      P.send_doubles += 15 * (int64_t)pe.send_cams.size() + 3 * (int64_t)pe.send_pts.size();
      P.recv_doubles += 15 * (int64_t)pe.recv_cams.size() + 3 * (int64_t)pe.recv_pts.size();
      P.peers.push_back(std::move(pe));
    }
  }
  return "";
}

bool order_owned_points(ShardPlan* S, const int32_t* obs_cam, bool force, int32_t far) {
  const int32_t np = S->n_own_pts;
  if (np < 2) return false;
  // key: smallest global camera observing the point (M if none)
  std::vector<int32_t> key((size_t)np);
  pfor(np, [&](int64_t a, int64_t b, int) {
    for (int64_t j = a; j < b; ++j) {
      int32_t m = (int32_t)S->M;
      for (int64_t q = S->pt_ptr[(size_t)j]; q < S->pt_ptr[(size_t)j + 1]; ++q)
        m = std::min(m, obs_cam[S->p_obs[(size_t)q]]);
      key[(size_t)j] = m;
    }
  });
  // keep a numbering that already follows the cameras: consecutive points whose smallest cameras lie far apart
  // (> 1024 camera ids) are rare in it (cluster changes), common in a scattered one
  std::atomic<int64_t> jumps(0);
  pfor(np - 1, [&](int64_t a, int64_t b, int) {
    int64_t d = 0;
    for (int64_t j = a; j < b; ++j) d += std::abs(key[(size_t)j + 1] - key[(size_t)j]) > far;
    jumps += d;
  });
  if (!force && jumps.load() * 4 < (int64_t)np) return false;
  // stable counting sort by key (owned points ascend by global id already)
  std::vector<int64_t> start((size_t)S->M + 2, 0);
  for (int32_t j = 0; j < np; ++j) ++start[(size_t)key[(size_t)j] + 1];
  for (size_t k = 1; k < start.size(); ++k) start[k] += start[k - 1];
  std::vector<int32_t> order((size_t)np), inv((size_t)np);
  for (int32_t j = 0; j < np; ++j) order[(size_t)start[(size_t)key[(size_t)j]]++] = j;
  pfor(np, [&](int64_t a, int64_t b, int) {
    for (int64_t q = a; q < b; ++q) inv[(size_t)order[(size_t)q]] = (int32_t)q;
  });
  {
    std::vector<int32_t> g((size_t)np);
    for (int32_t q = 0; q < np; ++q) g[(size_t)q] = S->pt_g[(size_t)order[(size_t)q]];
    std::copy(g.begin(), g.end(), S->pt_g.begin());
  }
  // camera side: new point ids, each camera's observations re-sorted by them (records of points with
  // neighbouring ids become neighbours)
  pfor(S->n_own_cams, [&](int64_t a, int64_t b, int) {
    std::vector<std::pair<int32_t, int32_t>> seg;
    for (int64_t i = a; i < b; ++i) {
      const int64_t lo = S->cam_ptr[(size_t)i], hi = S->cam_ptr[(size_t)i + 1];
      seg.clear();
      for (int64_t q = lo; q < hi; ++q) {
        const int32_t j = S->c_pt[(size_t)q];
        seg.emplace_back(j < np ? inv[(size_t)j] : j, S->c_obs[(size_t)q]);
      }
      std::sort(seg.begin(), seg.end());
      for (int64_t q = lo; q < hi; ++q) {
        S->c_pt[(size_t)q] = seg[(size_t)(q - lo)].first;
        S->c_obs[(size_t)q] = seg[(size_t)(q - lo)].second;
      }
    }
  }, (int64_t)S->c_obs.size());
  S->cam_side_identity = false;
  // point-side rows in the new order
  std::vector<int64_t> ptr((size_t)np + 1, 0);
  for (int32_t q = 0; q < np; ++q) {
    const int32_t j = order[(size_t)q];
    ptr[(size_t)q + 1] = ptr[(size_t)q] + (S->pt_ptr[(size_t)j + 1] - S->pt_ptr[(size_t)j]);
  }
  hvec<int32_t> pc(S->p_cam.size()), pp(S->p_pt.size()), po(S->p_obs.size());
  pfor(np, [&](int64_t a, int64_t b, int) {
    for (int64_t q = a; q < b; ++q) {
      const int32_t j = order[(size_t)q];
      int64_t d = ptr[(size_t)q];
      for (int64_t r = S->pt_ptr[(size_t)j]; r < S->pt_ptr[(size_t)j + 1]; ++r, ++d) {
        pc[(size_t)d] = S->p_cam[(size_t)r];
        pp[(size_t)d] = (int32_t)q;
        po[(size_t)d] = S->p_obs[(size_t)r];
      }
    }
  }, (int64_t)S->p_obs.size());
  S->pt_ptr.swap(ptr);
  S->p_cam.swap(pc);
  S->p_pt.swap(pp);
  S->p_obs.swap(po);
  for (Peer& pe : S->peers)
    for (int32_t& j : pe.send_pts) j = inv[(size_t)j];
  return true;
}

}  // namespace daba
