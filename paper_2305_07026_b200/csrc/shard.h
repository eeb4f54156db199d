// shard.h — host-side partition of a DABA problem across ranks (no CUDA).
//
// Partitioning follows P:L532 ("evenly distributing measurements to each device"): cameras in contiguous id
// ranges balanced by observation count; a point goes to the rank owning most of its observations (ties -> lowest
// rank).  Under reading D1 every observation is majorized, so the partition decides only what crosses the
// interconnect: rank r keeps
//   camera side: observations whose camera it owns (camera moments, F partial);
//   point side : observations whose point it owns (point sums);
//   halo       : non-owned points read by its camera side, non-owned cameras read by its point side,
// and exchanges x^k of boundary variables with its neighbours each iteration (Alg. 1).
#pragma once
#include <stdint.h>

#include <new>
#include <string>
#include <utility>
#include <vector>

namespace daba {

// Allocator whose value-less construct default-initialises (no zero fill): large host arrays are first touched
// by the parallel loops that fill them instead of by a serial memset.
template <class T>
struct NoInit : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInit<U>;
  };
  NoInit() = default;
  template <class U>
  NoInit(const NoInit<U>&) {}
  template <class U>
  void construct(U* p) noexcept {
    ::new ((void*)p) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new ((void*)p) U(std::forward<A>(a)...);
  }
};
template <class T>
using hvec = std::vector<T, NoInit<T>>;

struct Peer {
  int rank;
  std::vector<int32_t> send_cams, send_pts;  // LOCAL indices of owned entries to send (sorted by global id)
  std::vector<int32_t> recv_cams, recv_pts;  // LOCAL indices of halo slots to fill (sorted by global id)
};

struct ShardPlan {
  int rank = 0, nranks = 1;
  int64_t M = 0, N = 0, K = 0;
  std::vector<int32_t> cam_owner, pt_owner;     // global ownership maps
  std::vector<int32_t> cam_g, pt_g;             // local -> global ids: owned (ascending) then halo (ascending)
  int32_t n_own_cams = 0, n_own_pts = 0;
  // camera side (sorted by camera, then point): local camera, local point, global observation id
  hvec<int32_t> c_cam, c_pt;
  hvec<int32_t> c_obs;
  bool cam_side_identity = false;               // c_obs[q] = q (1 rank, input sorted by (camera, point))
  bool point_side_deferred = false;             // light plan: c_* and p_* not built (the engine builds the
                                                // point side on the device; identity camera side)
  std::vector<int64_t> cam_ptr;                 // n_own_cams + 1 offsets into the camera side
  // point side (sorted by point, then camera)
  hvec<int32_t> p_cam, p_pt;
  hvec<int32_t> p_obs;
  std::vector<int64_t> pt_ptr;                  // n_own_pts + 1
  std::vector<Peer> peers;
  int64_t send_doubles = 0, recv_doubles = 0;   // per iteration
};

// Renumber the owned points by (smallest observing camera id, global id) when the input numbering does not
// follow the cameras (a quarter or more of consecutive points have smallest cameras > 1024 ids apart), and
// re-sort each camera's observations by the new ids: points seen by the same cameras get neighbouring ids and
// their records neighbouring slots.  Measured on Final-13682 with randomly numbered points: point pass 1.17 ->
// 0.58 ms, camera pass 0.88 -> 0.76 ms, for ≈ 0.4 s more in daba_create.  The generator's host-camera numbering
// is kept (renumbering it would save 0.04 ms per iteration for the same create cost).  Returns whether it
// renumbered.
bool order_owned_points(ShardPlan* plan, const int32_t* obs_cam, bool force = false, int32_t far = 1024);

// Build rank `rank`'s shard.  cam_owner/pt_owner may be null (defaults above).  Returns "" or an error message
// (index out of range, duplicate (i,j), owner out of range).
// defer_point_side: with one rank and input sorted by (camera, point), stop after the camera offsets (a light
// plan, point_side_deferred) — the engine derives the rest on the device.
std::string plan_shard(int64_t M, int64_t N, int64_t K, const int32_t* obs_cam, const int32_t* obs_pt,
                       const int32_t* cam_owner, const int32_t* pt_owner, int rank, int nranks, ShardPlan* out,
                       bool defer_point_side = false);

// The light plan of one rank whose observations are sorted by (camera, point) (checked by the caller): identity
// numbering, every camera and point owned, camera offsets cam_ptr (M + 1); the point side is left to the engine.
void plan_light(int64_t M, int64_t N, int64_t K, std::vector<int64_t> cam_ptr, ShardPlan* out);

}  // namespace daba
