// kernels.h — launch interface of the DABA iteration kernels (host side).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace daba {

// Camera record in HBM: 16 doubles (128 B, one cache line): R[0..8] row-major camera->world, t[9..11] centre,
// d[12..14] = (f, f k1, f k2), [15] unused.
constexpr int kCamStride = 16;
constexpr int kNumMoments = 40;   // per camera and anchor, see DESIGN.md "camera moments"
constexpr int kPartialStride = 41;  // 40 moments + degenerate-pair count
#ifndef DABA_CPT
#define DABA_CPT 64  // one warp per anchor (k_cam_pass 0.741 ms on Final-13682)
#endif
constexpr int kCamPassThreads = DABA_CPT;  // threads per camera-pass CTA: half per anchor
constexpr int kCamWarps = kCamPassThreads / 32;
#ifndef DABA_CHUNK
#define DABA_CHUNK 4096
#endif
constexpr int kCamChunkObs = DABA_CHUNK;  // max observations per camera-pass chunk (one CTA)
constexpr int kPtPassThreads = 256;     // point solve: threads (points) per CTA
constexpr int kCamEvalCols = 8;   // F, dP_acc, dP_mm, step2_acc, step2_mm, ndeg, noacc_acc, noacc_mm
constexpr int kPtCols = 4;        // dQ_acc, dQ_mm, step2_acc, step2_mm
constexpr int kGlobalCols = 12;   // F, dP_acc, dQ_acc, dP_mm, dQ_mm, step2_acc, step2_mm, ndeg, noacc_acc, noacc_mm,
                                  // F_kappa correction, D increment (per-device restart, k_inter)
constexpr int kTraceCols = 11;    // = DABA_TRACE_COLS
constexpr int kInterThreads = 256;
// halo record of a camera: [acc 15 | mm 15 | acc x-bar 16 | mm x-bar 16] — the next iteration's x-bar travels
// with the state (the receiver would recompute the same ProjRot3D); of a point: [acc 3 | mm 3]
constexpr int kHaloCam = 62;

struct CamChunk {
  int32_t cam;    // local camera index (owned)
  int32_t n;      // observations in the chunk
  int64_t o0;     // first camera-side observation
};

// Device state of one iteration.  Role buffers: roles[0] = x^{k-1}, roles[1] = x^k, roles[2] = acc candidate,
// roles[3] = mm candidate; x-bar buffers (three per variable kind): roles[4] = x-bar^k, roles[5] / roles[6] =
// x-bar^{k+1} if the accelerated / MM candidate is selected.  The select kernel rotates them on the device, so
// that no kernel reading x-bar^k shares a buffer with one writing x-bar^{k+1} (the solves run beside each other).
struct IterParams {
  // sizes
  int32_t n_cams;        // local cameras (owned first, then halo)
  int32_t n_own_cams;
  int32_t n_pts;         // local points (owned first, then halo)
  int32_t n_own_pts;
  int32_t n_chunks;      // camera-pass chunks
  int32_t cam_shared_ctas;  // 1: one camera-pass CTA per chunk (both anchors), 0: one per chunk and anchor
  int32_t loss;
  double delta, delta2, idelta2;
  double xi, eta, mu0, mu_up, eps2;
  int32_t max_trials, accelerate;
  // state
  double* cams[4];       // n_cams x 16
  double4* pts[4];       // n_pts
  double4* lbar[3];      // x-bar of the points (roles[4..6])
  double* cbarb[3];      // x-bar of the cameras, n_cams x 16 (roles[4..6])
  int32_t* roles;        // [7]: x^{k-1}, x^k, acc, mm buffers; x-bar^k, x-bar^{k+1} (acc), x-bar^{k+1} (mm)
  double* sched;         // [0] s^{(k)}, [1] F-bar^{(k-1)}, [2] iteration counter k (as double)
  int32_t* counter;      // last-block detection of k_reduce (zero between launches)
  int32_t has_comm;      // 1: sums are allreduced, k_select runs after the collective
  // camera-side observations (sorted by camera, then point)
  const CamChunk* chunks;
  const int32_t* cam_chunk_ptr;  // n_own_cams + 1
  const double2* c_uv;
  const int32_t* c_pt;
  // point side: the camera pass writes, per camera-side observation o, the record (w lam^2, w lam R e) at
  // staging[o] (x-bar anchor) and staging[n_records + o] (x^k anchor), 4 doubles each; boundary observations
  // get records n_cam_side + b.  p_src lists each owned point's records in (point, camera) order.
  const int64_t* p_ptr;          // n_own_pts + 1
  const int32_t* p_src;          // record of each point-side observation
  double* staging;               // 2 x n_records x 4
  int64_t n_cam_side, n_records;
  // boundary observations (point owned here, camera owned elsewhere): recomputed from halo cameras
  int64_t n_boundary;
  const int32_t* b_cam;
  const int32_t* b_pt;
  const double2* b_uv;
  // scratch
  double* partial;        // n_chunks * 2 * kPartialStride
  double* moments;        // n_own_cams * 2 * kNumMoments (summed per camera)
  double* dP_mm;          // n_own_cams
  int32_t* decisions;     // n_own_cams * 2
  double* cam_part;       // camera-eval blocks x kCamEvalCols
  double* pt_part;        // point-pass blocks x kPtCols
  int32_t n_cam_eval_blocks, n_pt_blocks;
  double* local;          // kGlobalCols (this rank's sums)
  double* global;         // kGlobalCols (allreduced)
  double* trace;          // trace ring, trace_cap x kTraceCols
  int32_t trace_cap;
  // decentralized (per-device) restart, DABA_RESTART_DEVICE: the inter-device pairs this rank touches —
  // camera-side pairs with a halo point (sign +1) and point-side boundary pairs with a halo camera (sign -1)
  int32_t restart_scope;  // 0 global, 1 per device
  int64_t n_inter;
  const int32_t* i_cam;   // local camera
  const int32_t* i_pt;    // local point
  const double2* i_uv;
  const int32_t* i_sign;
  double* inter_part;     // k_inter blocks x 2
  int32_t n_inter_blocks;
  // halo send slots written by the solves themselves (global restart test with a communicator; no k_pack):
  // owned camera i / point j goes to send slots [ptr[i], ptr[i+1]), each at buffer offset off[s]
  double* sendbuf;        // null: a separate k_pack
  const int32_t* cam_send_ptr;
  const int64_t* cam_send_off;
  const int32_t* pt_send_ptr;
  const int64_t* pt_send_off;
};

// Launchers (all asynchronous on `st`).  They return the number of kernels launched.
int launch_lbar_all(const IterParams& p, cudaStream_t st);
int launch_cam_pass(const IterParams& p, cudaStream_t st);
int launch_pt_pass(const IterParams& p, cudaStream_t st);
int launch_cam_solve(const IterParams& p, cudaStream_t st);
int launch_pt_sum(const IterParams& p, cudaStream_t st);  // + rank-local sums (+ select without comm)
int launch_select(const IterParams& p, cudaStream_t st);
// per-device restart: the inter-device pair terms of F^{a(k)} (before k_cam_solve); rank-local sums of them
// into local[10..11] (create time); the allreduced trace columns after a local decision
int launch_inter(const IterParams& p, cudaStream_t st);
int launch_reduce_inter(const IterParams& p, cudaStream_t st);
int launch_trace_post(const IterParams& p, cudaStream_t st);
// F(x^k) only (create-time F-bar^{(-1)} and daba_objective): writes local[0] (and local[7] = degenerate count)
int launch_objective(const IterParams& p, cudaStream_t st);
// BAL pixel reprojection error of the state in role slot `role` (1: x^k, 0: x^{k-1}) over the camera-side
// observations: out[0..3] (device) = sum |r|, sum |r|^2, #(P'_z <= 0), #observations; resid (device, or null):
// |r| per camera-side observation
int launch_pixel_error(const IterParams& p, int role, double* out, double* resid, cudaStream_t st);
// halo exchange helpers: gather owned boundary entries of x^k into a send buffer / scatter received entries
// (selected = 1: after a local decision both slots carry x^{k+1})
int launch_pack(const IterParams& p, const int32_t* cam_idx, const int64_t* cam_off, int32_t n_cam,
                const int32_t* pt_idx, const int64_t* pt_off, int32_t n_pt, double* buf, int selected,
                cudaStream_t st);
// also writes x-bar of the received halo entries (gamma of the next iteration).  select_inside = 1: the
// restart decision is taken inside (every thread from the allreduced sums; the last block commits it), no
// separate k_select
int launch_unpack(const IterParams& p, const int32_t* cam_idx, const int64_t* cam_off, int32_t n_cam,
                  const int32_t* pt_idx, const int64_t* pt_off, int32_t n_pt, const double* buf, int select_inside,
                  cudaStream_t st);

// state readback: owned points as packed xyz (n x 3) in `dst` (device)
int launch_pts_xyz(const double4* src, double* dst, int32_t n, cudaStream_t st);
// and back: packed xyz (device) -> 32 B point records
int launch_xyz_pts(const double* src, double4* dst, int32_t n, cudaStream_t st);

// Create time, one rank with input sorted by (camera, point), from device copies of the observations' cameras
// and points: how many consecutive points have smallest observing cameras more than `far` ids apart (-1 on a
// CUDA error; shard.h order_owned_points), and the record list of every point in camera order (d_src, K: the
// observation index is the record index) with its offsets (d_ptr, N + 1; 0 or -1).
// (scratch: device memory for the temporaries — the record staging buffer, 64 B per observation, before its
// first use)
int64_t count_point_jumps_device(const int32_t* d_cam, const int32_t* d_pt, int64_t K, int32_t N, int32_t far,
                                 void* scratch, cudaStream_t st);
// Create time, one rank (device copies of the observations' cameras and points, K > 0): *bad_k = the first
// observation with an index out of range (K if none); *sorted = strictly sorted by (camera, point); when sorted and
// valid, cam_ptr_host (HOST, M + 1) = each camera's first observation.  scratch: 16 + 8 (M + 1) bytes + 512.
// 0 or -1 on a CUDA error.
int validate_sorted_device(const int32_t* d_cam, const int32_t* d_pt, int64_t K, int64_t M, int64_t N, void* scratch,
                           int64_t* bad_k, bool* sorted, int64_t* cam_ptr_host, cudaStream_t st);
int sort_point_side_device(const int32_t* d_pt, int64_t K, int32_t N, int32_t* d_src, int64_t* d_ptr, void* scratch,
                           size_t scratch_bytes, cudaStream_t st);

}  // namespace daba
