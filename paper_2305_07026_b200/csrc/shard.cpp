// shard.cpp — host-side partition and halo plan (see shard.h).
//
// Linear-time passes over the observations (counting sorts); the common case of input already sorted by
// (camera, point) skips the camera sort.
#include "shard.h"

#include <algorithm>
#include <cstdio>

namespace daba {

namespace {

// Stable counting sort of observation ids by key (0..nkeys-1); ptr gets nkeys+1 offsets.
void bucket(int64_t nkeys, const std::vector<int32_t>& ids, const int32_t* key, std::vector<int64_t>& ptr,
            std::vector<int32_t>& out) {
  ptr.assign((size_t)nkeys + 1, 0);
  for (int32_t o : ids) ++ptr[(size_t)key[o] + 1];
  for (int64_t k = 0; k < nkeys; ++k) ptr[(size_t)k + 1] += ptr[(size_t)k];
  out.resize(ids.size());
  std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
  for (int32_t o : ids) out[(size_t)pos[(size_t)key[o]]++] = o;
}

}  // namespace

std::string plan_shard(int64_t M, int64_t N, int64_t K, const int32_t* obs_cam, const int32_t* obs_pt,
                       const int32_t* cam_owner_in, const int32_t* pt_owner_in, int rank, int nranks,
                       ShardPlan* out) {
  char msg[256];
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
  bool sorted = true;  // by (camera, point), strictly
  for (int64_t k = 0; k < K; ++k) {
    if (obs_cam[k] < 0 || obs_cam[k] >= M || obs_pt[k] < 0 || obs_pt[k] >= N) {
      snprintf(msg, sizeof msg, "observation %lld has index out of range (camera %d, point %d)", (long long)k,
               obs_cam[k], obs_pt[k]);
      return msg;
    }
    if (k > 0 && sorted &&
        !(obs_cam[k - 1] < obs_cam[k] || (obs_cam[k - 1] == obs_cam[k] && obs_pt[k - 1] < obs_pt[k])))
      sorted = false;
  }
  // ---- observations in (camera, point) order; duplicate (i,j) check
  std::vector<int32_t> cam_sorted;
  std::vector<int64_t> cptr((size_t)M + 1, 0);
  if (sorted) {
    cam_sorted.resize((size_t)K);
    for (int64_t k = 0; k < K; ++k) {
      cam_sorted[(size_t)k] = (int32_t)k;
      ++cptr[(size_t)obs_cam[k] + 1];
    }
    for (int64_t i = 0; i < M; ++i) cptr[(size_t)i + 1] += cptr[(size_t)i];
  } else {
    std::vector<int32_t> all((size_t)K);
    for (int64_t k = 0; k < K; ++k) all[(size_t)k] = (int32_t)k;
    bucket(M, all, obs_cam, cptr, cam_sorted);
    for (int64_t i = 0; i < M; ++i) {
      auto b = cam_sorted.begin() + cptr[(size_t)i], e = cam_sorted.begin() + cptr[(size_t)i + 1];
      std::stable_sort(b, e, [&](int32_t x, int32_t y) { return obs_pt[x] < obs_pt[y]; });
      for (auto it = b; it + 1 < e; ++it)
        if (obs_pt[*(it + 1)] == obs_pt[*it]) {
          snprintf(msg, sizeof msg, "duplicate observation (camera %lld, point %d)", (long long)i, obs_pt[*it]);
          return msg;
        }
    }
  }
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
  // ---- point ownership (observations bucketed by point; stable, so cameras ascend within a point)
  std::vector<int32_t> pt_sorted;
  std::vector<int64_t> pptr;
  bucket(N, cam_sorted, obs_pt, pptr, pt_sorted);
  P.pt_owner.assign((size_t)N, 0);
  if (pt_owner_in) {
    for (int64_t j = 0; j < N; ++j) {
      if (pt_owner_in[j] < 0 || pt_owner_in[j] >= nranks) return "pt_owner entry out of range";
      P.pt_owner[(size_t)j] = pt_owner_in[j];
    }
  } else if (nranks > 1) {
    std::vector<int64_t> cnt((size_t)nranks);
    for (int64_t j = 0; j < N; ++j) {
      std::fill(cnt.begin(), cnt.end(), 0);
      for (int64_t q = pptr[(size_t)j]; q < pptr[(size_t)j + 1]; ++q)
        ++cnt[(size_t)P.cam_owner[(size_t)obs_cam[pt_sorted[(size_t)q]]]];
      int best = 0;
      for (int r = 1; r < nranks; ++r)
        if (cnt[(size_t)r] > cnt[(size_t)best]) best = r;  // ties -> lowest rank
      P.pt_owner[(size_t)j] = best;
    }
  }
  // ---- local numbering: owned first (ascending global id), halo after
  std::vector<int32_t> g2l_cam((size_t)M, -1), g2l_pt((size_t)N, -1);
  for (int64_t i = 0; i < M; ++i)
    if (P.cam_owner[(size_t)i] == rank) {
      g2l_cam[(size_t)i] = (int32_t)P.cam_g.size();
      P.cam_g.push_back((int32_t)i);
    }
  for (int64_t j = 0; j < N; ++j)
    if (P.pt_owner[(size_t)j] == rank) {
      g2l_pt[(size_t)j] = (int32_t)P.pt_g.size();
      P.pt_g.push_back((int32_t)j);
    }
  P.n_own_cams = (int32_t)P.cam_g.size();
  P.n_own_pts = (int32_t)P.pt_g.size();
  if (nranks > 1) {
    // halo points: read by the camera side; halo cameras: read by the point side
    std::vector<uint8_t> need_pt((size_t)N, 0), need_cam((size_t)M, 0);
    for (int32_t o : cam_sorted)
      if (P.cam_owner[(size_t)obs_cam[o]] == rank && P.pt_owner[(size_t)obs_pt[o]] != rank)
        need_pt[(size_t)obs_pt[o]] = 1;
    for (int32_t o : pt_sorted)
      if (P.pt_owner[(size_t)obs_pt[o]] == rank && P.cam_owner[(size_t)obs_cam[o]] != rank)
        need_cam[(size_t)obs_cam[o]] = 1;
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
  // ---- camera side, point side
  int64_t kc = 0, kp = 0;
  for (int32_t li = 0; li < P.n_own_cams; ++li) {
    const int64_t gi = P.cam_g[(size_t)li];
    kc += cptr[(size_t)gi + 1] - cptr[(size_t)gi];
  }
  for (int32_t lj = 0; lj < P.n_own_pts; ++lj) {
    const int64_t gj = P.pt_g[(size_t)lj];
    kp += pptr[(size_t)gj + 1] - pptr[(size_t)gj];
  }
  P.c_cam.resize((size_t)kc);
  P.c_pt.resize((size_t)kc);
  P.c_obs.resize((size_t)kc);
  P.cam_ptr.assign((size_t)P.n_own_cams + 1, 0);
  int64_t w = 0;
  for (int32_t li = 0; li < P.n_own_cams; ++li) {
    const int64_t gi = P.cam_g[(size_t)li];
    for (int64_t q = cptr[(size_t)gi]; q < cptr[(size_t)gi + 1]; ++q, ++w) {
      const int32_t o = cam_sorted[(size_t)q];
      P.c_cam[(size_t)w] = li;
      P.c_pt[(size_t)w] = g2l_pt[(size_t)obs_pt[o]];
      P.c_obs[(size_t)w] = o;
    }
    P.cam_ptr[(size_t)li + 1] = w;
  }
  P.p_cam.resize((size_t)kp);
  P.p_pt.resize((size_t)kp);
  P.p_obs.resize((size_t)kp);
  P.pt_ptr.assign((size_t)P.n_own_pts + 1, 0);
  w = 0;
  for (int32_t lj = 0; lj < P.n_own_pts; ++lj) {
    const int64_t gj = P.pt_g[(size_t)lj];
    for (int64_t q = pptr[(size_t)gj]; q < pptr[(size_t)gj + 1]; ++q, ++w) {
      const int32_t o = pt_sorted[(size_t)q];
      P.p_cam[(size_t)w] = g2l_cam[(size_t)obs_cam[o]];
      P.p_pt[(size_t)w] = lj;
      P.p_obs[(size_t)w] = o;
    }
    P.pt_ptr[(size_t)lj + 1] = w;
  }
  // ---- peers
  if (nranks > 1) {
    std::vector<std::vector<uint8_t>> sc((size_t)nranks, std::vector<uint8_t>((size_t)P.n_own_cams, 0));
    std::vector<std::vector<uint8_t>> sp((size_t)nranks, std::vector<uint8_t>((size_t)P.n_own_pts, 0));
    for (size_t q = 0; q < P.c_obs.size(); ++q) {
      const int b = P.pt_owner[(size_t)obs_pt[P.c_obs[q]]];
      if (b != rank) sc[(size_t)b][(size_t)P.c_cam[q]] = 1;
    }
    for (size_t q = 0; q < P.p_obs.size(); ++q) {
      const int b = P.cam_owner[(size_t)obs_cam[P.p_obs[q]]];
      if (b != rank) sp[(size_t)b][(size_t)P.p_pt[q]] = 1;
    }
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

}  // namespace daba
