// plan_api.cpp — host-only C-ABI over the shard planner (shard.h), for tests and tooling.
#include <cstring>
#include <new>

#include "../../include/daba.h"
#include "shard.h"

struct daba_plan {
  daba::ShardPlan S;
};

extern "C" daba_plan* daba_plan_create(int64_t M, int64_t N, const int32_t* obs_cam, const int32_t* obs_pt, int64_t K,
                                       const int32_t* cam_owner, const int32_t* pt_owner, int rank, int nranks) {
  daba_plan* p = new (std::nothrow) daba_plan();
  if (!p) return nullptr;
  if (!daba::plan_shard(M, N, K, obs_cam, obs_pt, cam_owner, pt_owner, rank, nranks, &p->S).empty()) {
    delete p;
    return nullptr;
  }
  return p;
}

extern "C" int daba_plan_counts(const daba_plan* p, int64_t c[10]) {
  if (!p || !c) return DABA_E_INVALID_ARG;
  const daba::ShardPlan& S = p->S;
  c[0] = S.n_own_cams;
  c[1] = S.n_own_pts;
  c[2] = (int64_t)S.cam_g.size() - S.n_own_cams;
  c[3] = (int64_t)S.pt_g.size() - S.n_own_pts;
  c[4] = (int64_t)S.c_obs.size();
  c[5] = (int64_t)S.p_obs.size();
  c[6] = S.send_doubles;
  c[7] = S.recv_doubles;
  c[8] = (int64_t)S.peers.size();
  c[9] = 0;
  return DABA_OK;
}

extern "C" int daba_plan_array(const daba_plan* p, int which, int32_t* out) {
  if (!p || !out) return DABA_E_INVALID_ARG;
  const daba::ShardPlan& S = p->S;
  const std::vector<int32_t>* v = nullptr;
  std::vector<int32_t> ranks;
  switch (which) {
    case 0: v = &S.cam_g; break;
    case 1: v = &S.pt_g; break;
    case 2: v = &S.cam_owner; break;
    case 3: v = &S.pt_owner; break;
    case 4:
      for (const daba::Peer& pe : S.peers) ranks.push_back(pe.rank);
      v = &ranks;
      break;
    default: return DABA_E_INVALID_ARG;
  }
  if (!v->empty()) std::memcpy(out, v->data(), v->size() * sizeof(int32_t));
  return DABA_OK;
}

extern "C" int64_t daba_plan_peer_list(const daba_plan* p, int peer, int kind, int32_t* out) {
  if (!p || peer < 0 || peer >= (int)p->S.peers.size() || kind < 0 || kind > 3) return DABA_E_INVALID_ARG;
  const daba::Peer& pe = p->S.peers[(size_t)peer];
  const std::vector<int32_t>& loc = kind == 0 ? pe.send_cams : kind == 1 ? pe.send_pts : kind == 2 ? pe.recv_cams
                                                                                                    : pe.recv_pts;
  const std::vector<int32_t>& g = (kind == 0 || kind == 2) ? p->S.cam_g : p->S.pt_g;
  if (out)
    for (size_t q = 0; q < loc.size(); ++q) out[q] = g[(size_t)loc[q]];
  return (int64_t)loc.size();
}

extern "C" void daba_plan_destroy(daba_plan* p) { delete p; }
