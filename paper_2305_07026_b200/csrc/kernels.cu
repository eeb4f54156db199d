// kernels.cu — fp64 CUDA kernels of one DABA iteration for sm_100a.
//
// Step map:
//   a4+a5  k_cam_pass       per observation, both anchors: ray (eq. ray), lambda (eq. gamma
//                           P:L222-224), error (eq. error), w and a (eqs. w, a P:L216-221);
//                           block-reduced into 40 per-camera moments (the camera part of eq. P); the point
//                           side of each pair emitted as a record (w lam^2, w lam R e)
//   a7     k_pt_sum         per point: adds its records, exact minimiser of sum_i Q_ij + xi/2 ||l - l_hat||^2
//                           (eq. Q, eq. Ealpha), the point part of E(x_acc|x^k) (eq. Eak
//                           P:L374-376), and x-bar^{k+1} of both candidates (eq. nesterov_l)
//          k_pt_boundary    records of observations whose camera lives on another rank (N > 1)
//   a6+a8  k_cam_solve      per camera and anchor: Gauss-Newton normal equations from the moments, one
//                           successful Levenberg-Marquardt step by Jacobi-scaled 9x9 Cholesky, the
//                           candidates' x-bar^{k+1} (eqs. nesterov_R/t/d, ProjRot3D eq. proj_rot3d
//                           P:L332-337), and the camera part of E(x_acc|x^k) and F(x^k)
//   a9     final_reduce     deterministic rank sums, in the last block of k_cam_solve / k_pt_sum (-> allreduce
//                           when nranks > 1)
//   a9+a10 do_select        F-bar (eq. lFak), restart test (Alg. 1), role rotation: in
//                           that last block without a communicator (or with the per-device test, k_inter adding
//                           the inter-device terms of eq. DEalpha), else after the allreduce in k_unpack (which
//                           also writes the received halo) or k_select
//          k_pack / k_unpack halo send / receive buffers (N > 1); k_lbar_all, k_objective at create / resume
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>

#include "kernels.h"
#include "device_math.cuh"

namespace daba {

// Bounds-check build (-DDABA_CHECK, build.py check=True): every index a kernel dereferences is checked against
// the size it indexes; a violation prints the kernel, the index and its bound and traps (a CUDA error the host
// reports).  The pool's compute-sanitizer is closed, so this is the memory-safety check of the GPU suite
// (tests run with DABA_LIB pointing at libdaba_check.so; profiles/r02_check_build_tests.log).
#ifdef DABA_CHECK
#define DCHECK(cond, what, idx, bound)                                                                      \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("DABA_CHECK %s: %s index %lld bound %lld (block %d thread %d)\n", __func__, what, (long long)(idx), \
             (long long)(bound), (int)blockIdx.x, (int)threadIdx.x);                                        \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define DCHECK(cond, what, idx, bound) \
  do {                                \
  } while (0)
#endif

__device__ __forceinline__ double sched_gamma(double s, int accelerate, double* s_next_out) {
  // eq. nesterov_scalar in Algorithm 1 line 407's order: s^{(k+1)} first, then gamma^{(k)}
  const double s_next = (sqrt(4.0 * s * s + 1.0) + 1.0) / 2.0;
  if (s_next_out) *s_next_out = s_next;
  return accelerate ? (s - 1.0) / s_next : 0.0;
}

// 256-bit global access (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256): one instruction per 32-byte record.  The
// load is not volatile (it may be scheduled freely); the store has no memory clobber: nobody reads a record in
// the kernel that writes it, so loads may move across it.
__device__ __forceinline__ double4 ld256(const double4* q) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(q));
  return v;
}
// The same for gathers with no reuse in L1 (points by the camera pass, records by the point sums): no L1 line
// allocated, so the L1 / shared-memory array keeps what is reused (Final-13682: camera pass 0.704 -> 0.678 ms,
// point sums 0.590 -> 0.581 ms, iteration 1.309 -> 1.268 ms).
__device__ __forceinline__ double4 ld256_na(const double4* q) {
  double4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(q));
  return v;
}

__device__ __forceinline__ void st256(double4* q, double4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(q), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w));
}

// Point-side record of observation r at anchor a (0: x-bar^k, 1: x^k), 32 B, in two separate arrays.  (The two
// anchors' records side by side, 64 B: with one CTA per chunk and anchor k_pt_sum -0.04 / k_cam_pass +0.03 ms;
// with both anchors in one CTA k_pt_sum +0.025 / k_cam_pass +0.033 ms.)
__device__ __forceinline__ double4* rec_ptr(const IterParams& p, int64_t r, int a) {
  return reinterpret_cast<double4*>(p.staging + (a ? 4 * p.n_records : 0)) + r;
}

// Point record: 32 bytes (x, y, z, pad) — one sector per gather.
__device__ __forceinline__ void ld_point(const double4* base, int64_t j, double& x, double& y, double& z) {
  const double2* q = reinterpret_cast<const double2*>(base + j);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  x = a.x;
  y = a.y;
  z = b.x;
}

// gamma^{(k+1)} from s^{(k)} (two schedule steps), for the x-bar of the next iteration
__device__ __forceinline__ double sched_gamma_next(double s, int accelerate) {
  double s1;
  sched_gamma(s, accelerate, &s1);
  return sched_gamma(s1, accelerate, nullptr);
}

// x-bar camera (eqs. nesterov_R/t/d): ProjRot3D(R + g (R - R_prev)), t, d linear
__device__ __forceinline__ void extrapolate_camera(const double* ck, const double* cp, double gamma, double* out) {
  double M[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) M[k] = ck[k] + gamma * (ck[k] - cp[k]);
  proj_rot3d(M, out);
#pragma unroll
  for (int k = 9; k < 15; ++k) out[k] = ck[k] + gamma * (ck[k] - cp[k]);
  out[15] = 0.0;
}

// ------------------------------------------------------------------ a4 + a5: camera pass
// Moment slots (anchor camera frame; e = camera-frame reprojection error, s = |u|^2):
//  0 w ux^2   1 w ux uy  2 w uy^2   3-5 w ux s^m  6-8 w uy s^m  9-13 w s^m (m=0..4)
//  14 w lam ux  15 w lam uy  16-18 w lam s^m  19 w lam^2
//  20-22 w e ux  23-25 w e uy  26-28 w e  29-31 w e s  32-34 w e s^2  35-37 w lam e   (e = R e, world frame;
//        k_cam_solve rotates them into the anchor camera frame: the camera pass never applies R^T)
//  38 (unused: 0)   39 rho / 2 = a + w |e|^2 / 2   [40 degenerate pairs]
// Camera record kept in shared memory and re-read at every use (volatile shared loads are not hoisted into
// registers): frees ~30 registers per thread in the camera pass, i.e. more resident CTAs per SM (a copy in
// registers measured 0.80 ms with spills at 6 CTAs/SM, 0.86 ms at 4).
struct CamRegs {
  const double* sm;  // shared-memory camera record (16 doubles)
  __device__ __forceinline__ double operator[](int k) const {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(sm + k)));
    return v;
  }
};
#ifndef DABA_RING
#define DABA_RING 8
#endif
#ifndef DABA_MINB
#define DABA_MINB (384 / DABA_CPT)  // 12 warps per SM: the 170-register budget of the moment accumulators
#endif

// One observation's moments and point-side record at one anchor, from its geometry (s = |u|^2, lambda, the
// world-frame error R e, |R e|^2, w = rho', rho).
template <bool ACC>
__device__ __forceinline__ void obs_moments(const IterParams& p, double2 u, double s, double s2, double lam, double ex,
                                            double ey, double ez, double sh, double w, double rho, double* acc,
                                            int64_t rec) {
  const double wx = w * u.x, wy = w * u.y, ws = w * s, ws2 = w * s2;
  acc[0] = fma(wx, u.x, acc[0]);
  acc[1] = fma(wx, u.y, acc[1]);
  acc[2] = fma(wy, u.y, acc[2]);
  acc[3] += wx;
  acc[4] = fma(wx, s, acc[4]);
  acc[5] = fma(wx, s2, acc[5]);
  acc[6] += wy;
  acc[7] = fma(wy, s, acc[7]);
  acc[8] = fma(wy, s2, acc[8]);
  acc[9] += w;
  acc[10] += ws;
  acc[11] += ws2;
  acc[12] = fma(ws2, s, acc[12]);
  acc[13] = fma(ws2, s2, acc[13]);
  const double wl = w * lam;
  acc[14] = fma(wl, u.x, acc[14]);
  acc[15] = fma(wl, u.y, acc[15]);
  acc[16] += wl;
  acc[17] = fma(wl, s, acc[17]);
  acc[18] = fma(wl, s2, acc[18]);
  acc[19] = fma(wl, lam, acc[19]);
  // error moments from the weighted factors already formed (w u_x, w u_y, w, w s, w s^2, w lam): one FMA each
  acc[20] = fma(wx, ex, acc[20]);
  acc[21] = fma(wx, ey, acc[21]);
  acc[22] = fma(wx, ez, acc[22]);
  acc[23] = fma(wy, ex, acc[23]);
  acc[24] = fma(wy, ey, acc[24]);
  acc[25] = fma(wy, ez, acc[25]);
  acc[26] = fma(w, ex, acc[26]);
  acc[27] = fma(w, ey, acc[27]);
  acc[28] = fma(w, ez, acc[28]);
  acc[29] = fma(ws, ex, acc[29]);
  acc[30] = fma(ws, ey, acc[30]);
  acc[31] = fma(ws, ez, acc[31]);
  acc[32] = fma(ws2, ex, acc[32]);
  acc[33] = fma(ws2, ey, acc[33]);
  acc[34] = fma(ws2, ez, acc[34]);
  acc[35] = fma(wl, ex, acc[35]);
  acc[36] = fma(wl, ey, acc[36]);
  acc[37] = fma(wl, ez, acc[37]);
  if (!ACC)  // F_i = sum (a + w |e|^2 / 2) = sum rho / 2 (eqs. a, Fij): one accumulator (slot 38 stays 0)
    acc[39] = fma(0.5, rho, acc[39]);
  // point side of the same pair: (w lam^2, w lam R e) with the world-frame error R e (eq. Q's sums), written
  // coalesced at the camera-side index (one 32-byte record per anchor)
  if (rec >= 0)
    st256(rec_ptr(p, rec, ACC ? 0 : 1), make_double4(wl * lam, wl * ex, wl * ey, wl * ez));
}

// Two observations of one camera at one anchor: each camera value is read from shared memory once for both
// (15 shared loads per pair instead of per observation), the two dependency chains interleaved.  Per observation:
// s = |u|^2, p = (u, d1 + d2 s + d3 s^2) (eq. ray), v = l - t, the world-frame ray R p, lambda = v.R p / |v|^2
// (eq. gamma), the world-frame error R e = R p - lambda v (eq. error; its moments are rotated into the anchor
// camera frame once per camera by k_cam_solve), w = rho'(|R e|^2) (eq. w); a pair violating Assumption 2 at this
// anchor contributes nothing (counted in slot 40, zero record).
template <int LOSS, bool ACC>
__device__ __forceinline__ void cam_obs2(const IterParams& p, const CamRegs& c, double2 u0, double4 l0, double2 u1,
                                         double4 l1, bool has1, double* acc, int64_t rec0, int64_t rec1) {
  const double s0 = fma(u0.x, u0.x, u0.y * u0.y), s1 = fma(u1.x, u1.x, u1.y * u1.y);
  double pz0, pz1, vx0, vy0, vz0, vx1, vy1, vz1, rx0, ry0, rz0, rx1, ry1, rz1;
  {
    const double d0 = c[12], d1 = c[13], d2 = c[14];
    pz0 = fma(s0, fma(s0, d2, d1), d0);  // eq. ray
    pz1 = fma(s1, fma(s1, d2, d1), d0);
  }
  {
    const double tx = c[9], ty = c[10], tz = c[11];
    vx0 = l0.x - tx; vy0 = l0.y - ty; vz0 = l0.z - tz;
    vx1 = l1.x - tx; vy1 = l1.y - ty; vz1 = l1.z - tz;
  }
  {
    const double a = c[0], b = c[1], d = c[2];
    rx0 = fma(a, u0.x, fma(b, u0.y, d * pz0));
    rx1 = fma(a, u1.x, fma(b, u1.y, d * pz1));
  }
  {
    const double a = c[3], b = c[4], d = c[5];
    ry0 = fma(a, u0.x, fma(b, u0.y, d * pz0));
    ry1 = fma(a, u1.x, fma(b, u1.y, d * pz1));
  }
  {
    const double a = c[6], b = c[7], d = c[8];
    rz0 = fma(a, u0.x, fma(b, u0.y, d * pz0));
    rz1 = fma(a, u1.x, fma(b, u1.y, d * pz1));
  }
  const double nv0 = fma(vx0, vx0, fma(vy0, vy0, vz0 * vz0)), nv1 = fma(vx1, vx1, fma(vy1, vy1, vz1 * vz1));
  const bool ok0 = nv0 > p.eps2, ok1 = nv1 > p.eps2;  // Assumption 2 at this anchor
  const double lam0 = fma(vx0, rx0, fma(vy0, ry0, vz0 * rz0)) * rcp_d(nv0);  // eq. gamma
  const double lam1 = fma(vx1, rx1, fma(vy1, ry1, vz1 * rz1)) * rcp_d(nv1);
  const double ex0 = fma(-lam0, vx0, rx0), ey0 = fma(-lam0, vy0, ry0), ez0 = fma(-lam0, vz0, rz0);  // eq. error
  const double ex1 = fma(-lam1, vx1, rx1), ey1 = fma(-lam1, vy1, ry1), ez1 = fma(-lam1, vz1, rz1);
  const double sh0 = fma(ex0, ex0, fma(ey0, ey0, ez0 * ez0)), sh1 = fma(ex1, ex1, fma(ey1, ey1, ez1 * ez1));
  if (ok0) {
    double rho = 0;
    const double w = loss_eval<LOSS, !ACC>(sh0, p.delta, p.delta2, p.idelta2, &rho);  // eq. w
    obs_moments<ACC>(p, u0, s0, s0 * s0, lam0, ex0, ey0, ez0, sh0, w, rho, acc, rec0);
  } else {  // the pair contributes nothing
    acc[40] += 1.0;
    if (rec0 >= 0) st256(rec_ptr(p, rec0, ACC ? 0 : 1), make_double4(0.0, 0.0, 0.0, 0.0));
  }
  if (!has1) return;
  if (ok1) {
    double rho = 0;
    const double w = loss_eval<LOSS, !ACC>(sh1, p.delta, p.delta2, p.idelta2, &rho);
    obs_moments<ACC>(p, u1, s1, s1 * s1, lam1, ex1, ey1, ez1, sh1, w, rho, acc, rec1);
  } else {
    acc[40] += 1.0;
    if (rec1 >= 0) st256(rec_ptr(p, rec1, ACC ? 0 : 1), make_double4(0.0, 0.0, 0.0, 0.0));
  }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Camera-pass streaming: u (coalesced) goes through a per-thread cp.async ring; the anchor point record
// (x-bar^k for the accelerated anchor, x^k for the MM anchor; 32 B) is gathered with one 256-bit load,
// prefetched one observation ahead in registers.  The chunk's point indices are staged in shared memory.
constexpr int kRing = DABA_RING;

// The chunk's point indices staged in shared memory (every 4-byte copy in flight at once, one wait) and the
// anchor camera's record; the caller synchronises the CTA afterwards.
__device__ __forceinline__ void stage_chunk(const IterParams& p, const CamChunk ch, int32_t* sidx) {
  for (int o = threadIdx.x; o < ch.n; o += kCamPassThreads) cp_async4(sidx + o, p.c_pt + ch.o0 + o);
  cp_async_commit();
  cp_async_wait<0>();
}

// One anchor's pass over a chunk by a group of G threads (lane = rank in the group): observation lane + G k.
template <int LOSS, bool ACC, int G>
__device__ __forceinline__ void cam_pass_body(const IterParams& p, const CamChunk ch, double* acc,
                                              double2* ring, const int32_t* sidx, int lane, const double* scam) {
  CamRegs c{scam};
  const double4* __restrict__ L = ACC ? p.lbar[p.roles[4]] : p.pts[p.roles[1]];
  const int tid = threadIdx.x;
  const int n = (ch.n - lane + G - 1) / G;  // observations of this thread
#define REC(kk) (ch.o0 + lane + (int64_t)(kk) * G)
  auto uslot = [&](int k) { return ring + (k & (kRing - 1)) * kCamPassThreads + tid; };
  auto issue = [&](int k) {
    if (k < n) cp_async16(uslot(k), p.c_uv + ch.o0 + lane + (int64_t)k * G);
    cp_async_commit();
  };
#pragma unroll
  for (int k = 0; k < kRing - 1; ++k) issue(k);
  // two observations per step: two independent dependency chains feed the same accumulators; the next step's
  // point records are in flight (registers).  (Measured: one observation per step 0.90 ms vs 0.76 ms; a deeper
  // record prefetch was slower.)
  double4 lq0 = 0 < n ? ld256_na(L + sidx[lane]) : make_double4(0, 0, 0, 0);
  double4 lq1 = 1 < n ? ld256_na(L + sidx[lane + G]) : make_double4(0, 0, 0, 0);
  issue(kRing - 1);
#pragma unroll 1
  for (int k = 0; k < n; k += 2) {
    const double4 l0 = lq0, l1 = lq1;
    if (k + 2 < n) lq0 = ld256_na(L + sidx[lane + (k + 2) * G]);
    if (k + 3 < n) lq1 = ld256_na(L + sidx[lane + (k + 3) * G]);
    cp_async_wait<kRing - 2>();  // groups k and k + 1 have landed
    const double2 u0 = *uslot(k);
    const double2 u1 = *uslot(k + 1);
    issue(k + kRing);  // refills the two slots just read
    issue(k + kRing + 1);
    // (one camera read per pair: 0.7093 -> 0.7034 ms against one observation at a time, Final-13682)
    cam_obs2<LOSS, ACC>(p, c, u0, l0, u1, l1, k + 1 < n, acc, REC(k), REC(k + 1));
  }
  cp_async_wait<0>();
#undef REC
}

// The moments of each group of G threads (the anchors of a CTA) summed in a fixed order via a shared-memory
// transpose; group g's sums go to out + g * kPartialStride.
template <int G>
__device__ __forceinline__ void group_reduce_moments(double* acc, double* out, double* smem) {
  double(*red)[32][kPartialStride] = reinterpret_cast<double(*)[32][kPartialStride]>(smem);
  __shared__ double wsum[kCamWarps][kPartialStride];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kPartialStride; ++k) red[warp][lane][k] = acc[k];
  __syncwarp();
  for (int k = lane; k < kPartialStride; k += 32) {
    double s0 = 0, s1 = 0;
#pragma unroll 4
    for (int r = 0; r < 32; r += 2) {
      s0 += red[warp][r][k];
      s1 += red[warp][r + 1][k];
    }
    wsum[warp][k] = s0 + s1;
  }
  constexpr int WG = G / 32, NG = kCamPassThreads / G;  // warps per group, groups
  if (WG == 1) {
    for (int k = lane; k < kPartialStride; k += 32) out[(size_t)warp * kPartialStride + k] = wsum[warp][k];
    return;
  }
  __syncthreads();
  if (threadIdx.x < NG * kPartialStride) {
    const int g = threadIdx.x / kPartialStride, k = threadIdx.x % kPartialStride;
    double v = 0.0;
    for (int w = 0; w < WG; ++w) v += wsum[g * WG + w][k];
    out[(size_t)g * kPartialStride + k] = v;
  }
}

constexpr int kCamRingDoubles = kRing * 2 * kCamPassThreads + kCamChunkObs / 2;  // ring + indices
constexpr int kCamSmemDoubles =
    kCamRingDoubles > kCamPassThreads * kPartialStride ? kCamRingDoubles : kCamPassThreads * kPartialStride;

// SHARED: one CTA per chunk, the first half of the threads the accelerated anchor and the second half the MM
// anchor, sharing the staged indices (large shards).  Otherwise one CTA per chunk and anchor, all threads on
// one anchor: twice the CTAs, for shards too small to fill the GPU a few times over (measured: Final-13682 at
// one rank 0.741 vs 0.764 ms; one rank of eight 0.247 vs 0.251 ms per iteration).
template <int LOSS, bool SHARED>
__global__ void __launch_bounds__(kCamPassThreads, DABA_MINB) k_cam_pass(IterParams p) {
  extern __shared__ __align__(16) double smem[];  // kCamSmemDoubles
  constexpr int G = SHARED ? kCamPassThreads / 2 : kCamPassThreads;
  const int chunk = SHARED ? blockIdx.x : blockIdx.x >> 1;
  const int grp = SHARED ? threadIdx.x / G : (blockIdx.x & 1), lane = threadIdx.x % G;
  DCHECK(chunk < p.n_chunks, "chunk", chunk, p.n_chunks);
  const CamChunk ch = p.chunks[chunk];
  DCHECK(ch.o0 >= 0 && ch.n <= kCamChunkObs && ch.o0 + ch.n <= p.n_cam_side, "chunk obs", ch.o0 + ch.n, p.n_cam_side);
  DCHECK(ch.cam >= 0 && ch.cam < p.n_own_cams, "chunk camera", ch.cam, p.n_own_cams);
  double acc[kPartialStride];
#pragma unroll
  for (int k = 0; k < kPartialStride; ++k) acc[k] = 0.0;
  double2* ring = reinterpret_cast<double2*>(smem);
  int32_t* sidx = reinterpret_cast<int32_t*>(smem + kRing * 2 * kCamPassThreads);
  __shared__ double scam[2][kCamStride];
  if (lane < kCamStride)
    scam[grp][lane] = (grp == 0 ? p.cbarb[p.roles[4]] : p.cams[p.roles[1]])[(size_t)ch.cam * kCamStride + lane];
  stage_chunk(p, ch, sidx);
#ifdef DABA_CHECK
  for (int o = threadIdx.x; o < ch.n; o += kCamPassThreads)
    DCHECK(sidx[o] >= 0 && sidx[o] < p.n_pts, "point", sidx[o], p.n_pts);
  DCHECK(ch.o0 + ch.n <= p.n_records, "record", ch.o0 + ch.n, p.n_records);
#endif
  __syncthreads();
  if (grp == 0)
    cam_pass_body<LOSS, true, G>(p, ch, acc, ring, sidx, lane, scam[0]);
  else
    cam_pass_body<LOSS, false, G>(p, ch, acc, ring, sidx, lane, scam[1]);
  __syncthreads();  // the ring is reused as the reduction buffer
  group_reduce_moments<G>(acc, p.partial + (size_t)(SHARED ? 2 * blockIdx.x : blockIdx.x) * kPartialStride, smem);
}

// ------------------------------------------------------------------ objective F(x^k) only
template <int LOSS>
__global__ void __launch_bounds__(kCamPassThreads) k_objective(IterParams p) {
  const CamChunk ch = p.chunks[blockIdx.x];
  const double* cam = p.cams[p.roles[1]] + (size_t)ch.cam * kCamStride;
  const double4* __restrict__ Lk = p.pts[p.roles[1]];
  double F = 0, nd = 0;
  for (int64_t o = ch.o0 + threadIdx.x; o < ch.o0 + ch.n; o += kCamPassThreads) {
    const int32_t j = p.c_pt[o];
    const double2 u = p.c_uv[o];
    const double4 l = Lk[j];
    const double s = fma(u.x, u.x, u.y * u.y);
    const double pz = fma(s, fma(s, cam[14], cam[13]), cam[12]);
    const double vx = l.x - cam[9], vy = l.y - cam[10], vz = l.z - cam[11];
    const double nv = fma(vx, vx, fma(vy, vy, vz * vz));
    if (!(nv > p.eps2)) {
      nd += 1.0;
      continue;
    }
    const double cx = fma(cam[0], vx, fma(cam[3], vy, cam[6] * vz));
    const double cy = fma(cam[1], vx, fma(cam[4], vy, cam[7] * vz));
    const double cz = fma(cam[2], vx, fma(cam[5], vy, cam[8] * vz));
    const double lam = fma(cx, u.x, fma(cy, u.y, cz * pz)) * __drcp_rn(nv);
    const double ex = fma(-lam, cx, u.x), ey = fma(-lam, cy, u.y), ez = fma(-lam, cz, pz);
    double rho;
    loss_eval<LOSS, true>(fma(ex, ex, fma(ey, ey, ez * ez)), p.delta, p.delta2, p.idelta2, &rho);
    F += 0.5 * rho;  // eq. Fij
  }
  __shared__ double sF[kCamPassThreads], sN[kCamPassThreads];
  sF[threadIdx.x] = F;
  sN[threadIdx.x] = nd;
  __syncthreads();
  for (int st = kCamPassThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      sF[threadIdx.x] += sF[threadIdx.x + st];
      sN[threadIdx.x] += sN[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.partial[(size_t)blockIdx.x * 2 * kPartialStride] = sF[0];
    p.partial[(size_t)blockIdx.x * 2 * kPartialStride + 1] = sN[0];
  }
}

__global__ void k_reduce_objective(IterParams p) {
  __shared__ double sF[256], sN[256];
  double F = 0, nd = 0;
  for (int c = threadIdx.x; c < p.n_chunks; c += 256) {
    F += p.partial[(size_t)c * 2 * kPartialStride];
    nd += p.partial[(size_t)c * 2 * kPartialStride + 1];
  }
  sF[threadIdx.x] = F;
  sN[threadIdx.x] = nd;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      sF[threadIdx.x] += sF[threadIdx.x + st];
      sN[threadIdx.x] += sN[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < kGlobalCols; ++k) p.local[k] = 0.0;
    p.local[0] = sF[0];
    p.local[7] = sN[0];
  }
}

// ------------------------------------------------------------------ pixel metric
// Mean reprojection error in pixels under the BAL forward model (the metric of Table 2), evaluated in
// the paper's frame: P' = R^T (l - t) (= S P_BAL with S = diag(1,-1,-1), see daba_bal_to_paper), q = P'_xy / P'_z,
// predicted u = f (1 + k1 |q|^2 + k2 |q|^4) q with BAL's k1 = f d2, k2 = f^3 d3 + 2 k1^2 (the inverse of the
// series reversion of the intrinsics), residual against the stored (v-flipped) observation.  Per chunk:
// [sum |r|, sum |r|^2, #(P'_z <= 0), #observations].
// |r| of one observation (pixels) and whether the point is behind the camera (P'_z <= 0)
__device__ __forceinline__ double pixel_residual(const double* cam, double f, double k1, double k2, double4 l,
                                                 double2 u, bool* behind) {
  const double vx = l.x - cam[9], vy = l.y - cam[10], vz = l.z - cam[11];
  const double cx = fma(cam[0], vx, fma(cam[3], vy, cam[6] * vz));
  const double cy = fma(cam[1], vx, fma(cam[4], vy, cam[7] * vz));
  const double cz = fma(cam[2], vx, fma(cam[5], vy, cam[8] * vz));
  *behind = cz <= 0.0;
  const double qx = cx / cz, qy = cy / cz;
  const double q2 = fma(qx, qx, qy * qy);
  const double g = f * fma(q2, fma(q2, k2, k1), 1.0);
  const double rx = fma(-g, qx, u.x), ry = fma(-g, qy, u.y);
  return sqrt(fma(rx, rx, ry * ry));
}

__global__ void __launch_bounds__(kCamPassThreads) k_pixel_error(IterParams p, int role, double* resid) {
  const CamChunk ch = p.chunks[blockIdx.x];
  const int r = p.roles[role];
  const double* cam = p.cams[r] + (size_t)ch.cam * kCamStride;
  const double4* __restrict__ L = p.pts[r];
  const double f = cam[12], k1 = f * cam[13], k2 = fma(f * f * f, cam[14], 2.0 * k1 * k1);
  double se = 0, se2 = 0, nb = 0;
  for (int64_t o = ch.o0 + threadIdx.x; o < ch.o0 + ch.n; o += kCamPassThreads) {
    bool behind;
    const double e = pixel_residual(cam, f, k1, k2, L[p.c_pt[o]], p.c_uv[o], &behind);
    nb += behind ? 1.0 : 0.0;
    se += e;
    se2 = fma(e, e, se2);
    if (resid) resid[o] = e;
  }
  __shared__ double sh[3][kCamPassThreads];
  sh[0][threadIdx.x] = se;
  sh[1][threadIdx.x] = se2;
  sh[2][threadIdx.x] = nb;
  __syncthreads();
  for (int st = kCamPassThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < 3; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* q = p.partial + (size_t)blockIdx.x * 2 * kPartialStride;
    q[0] = sh[0][0];
    q[1] = sh[1][0];
    q[2] = sh[2][0];
    q[3] = (double)ch.n;
  }
}

__global__ void k_reduce_pixel_error(IterParams p, double* out) {
  __shared__ double sh[4][256];
  double a[4] = {0, 0, 0, 0};
  for (int c = threadIdx.x; c < p.n_chunks; c += 256)
    for (int k = 0; k < 4; ++k) a[k] += p.partial[(size_t)c * 2 * kPartialStride + k];
  for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] = a[k];
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x < 4) out[threadIdx.x] = sh[threadIdx.x][0];
}

// ------------------------------------------------------------------ a4 + a5 + a7: point pass
template <int LOSS>
__device__ __forceinline__ void pt_terms(const double* cam, double lx, double ly, double lz, double2 u,
                                         const IterParams& p, double& A, double& Cx, double& Cy, double& Cz) {
  const double s = fma(u.x, u.x, u.y * u.y);
  const double pz = fma(s, fma(s, cam[14], cam[13]), cam[12]);  // eq. ray
  // world-frame ray R p
  const double rx = fma(cam[0], u.x, fma(cam[1], u.y, cam[2] * pz));
  const double ry = fma(cam[3], u.x, fma(cam[4], u.y, cam[5] * pz));
  const double rz = fma(cam[6], u.x, fma(cam[7], u.y, cam[8] * pz));
  const double vx = lx - cam[9], vy = ly - cam[10], vz = lz - cam[11];
  const double nv = fma(vx, vx, fma(vy, vy, vz * vz));
  if (!(nv > p.eps2)) return;
  const double lam = fma(vx, rx, fma(vy, ry, vz * rz)) * rcp_d(nv);  // eq. gamma
  const double ex = fma(-lam, vx, rx), ey = fma(-lam, vy, ry), ez = fma(-lam, vz, rz);  // R e (eq. error)
  const double w = loss_eval<LOSS, false>(fma(ex, ex, fma(ey, ey, ez * ez)), p.delta, p.delta2, p.idelta2, nullptr);
  const double wl = w * lam;
  A = fma(wl, lam, A);
  Cx = fma(wl, ex, Cx);
  Cy = fma(wl, ey, Cy);
  Cz = fma(wl, ez, Cz);
}

// Solve both anchors' point subproblems from their sums and write the candidates; returns the Q-part of
// E(x_acc|x^k) - E(x^k|x^k), of E(x_mm|x^k) - E(x^k|x^k), and the squared moves (q[0..3]).
__device__ __forceinline__ void pt_finish(const IterParams& p, int j, const double* lb, const double* lk,
                                          const double* a, double* q) {
  // exact minimiser: (2 A + xi) dl = C  (eq. Q with the proximal term of eq. Ealpha)
  const double ib = 1.0 / fma(2.0, a[0], p.xi), ik = 1.0 / fma(2.0, a[4], p.xi);
  const double ax = fma(a[1], ib, lb[0]), ay = fma(a[2], ib, lb[1]), az = fma(a[3], ib, lb[2]);  // l_acc
  const double mx = a[5] * ik, my = a[6] * ik, mz = a[7] * ik;                                  // l_mm - l^k
  p.pts[p.roles[2]][j] = make_double4(ax, ay, az, 0.0);
  const double nx = lk[0] + mx, ny = lk[1] + my, nz = lk[2] + mz;
  p.pts[p.roles[3]][j] = make_double4(nx, ny, nz, 0.0);
  // x-bar^{k+1} for either outcome of the restart test (eq. nesterov_l with gamma^{(k+1)}); k_select keeps one
  if (p.sendbuf)  // boundary point: both candidates straight into its halo send slots
    for (int s = p.pt_send_ptr[j]; s < p.pt_send_ptr[j + 1]; ++s) {
      double* b = p.sendbuf + p.pt_send_off[s];
      b[0] = ax;
      b[1] = ay;
      b[2] = az;
      b[3] = nx;
      b[4] = ny;
      b[5] = nz;
    }
  const double g1 = sched_gamma_next(p.sched[0], p.accelerate);
  p.lbar[p.roles[5]][j] = make_double4(fma(g1, ax - lk[0], ax), fma(g1, ay - lk[1], ay), fma(g1, az - lk[2], az), 0.0);
  p.lbar[p.roles[6]][j] = make_double4(fma(g1, nx - lk[0], nx), fma(g1, ny - lk[1], ny), fma(g1, nz - lk[2], nz), 0.0);
  // Q-part of E(x|x^k) - E(x^k|x^k): (A_k + xi/2) |dl|^2 - C_k . dl  (eq. Q expanded at the anchor)
  const double dx = ax - lk[0], dy = ay - lk[1], dz = az - lk[2];
  const double n_acc = fma(dx, dx, fma(dy, dy, dz * dz));
  const double n_mm = fma(mx, mx, fma(my, my, mz * mz));
  const double hk = fma(0.5, p.xi, a[4]);
  q[0] = fma(hk, n_acc, -fma(a[5], dx, fma(a[6], dy, a[7] * dz)));
  q[1] = fma(hk, n_mm, -fma(a[5], mx, fma(a[6], my, a[7] * mz)));
  q[2] = n_acc;
  q[3] = n_mm;
}

// Boundary observations (their camera is owned by another rank, N > 1 only): recompute the point-side
// contribution from the halo camera and write it into the staging record, like the camera pass does.
// A 128-byte camera record into registers: four 256-bit loads, all in flight together.
__device__ __forceinline__ void load_cam16(const double* c, double* out) {
  const double4* q = reinterpret_cast<const double4*>(c);
  double4 v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = ld256(q + k);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    out[4 * k] = v[k].x;
    out[4 * k + 1] = v[k].y;
    out[4 * k + 2] = v[k].z;
    out[4 * k + 3] = v[k].w;
  }
}

template <int LOSS>
__global__ void __launch_bounds__(256) k_pt_boundary(IterParams p) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= p.n_boundary) return;
  const int32_t i = p.b_cam[b], j = p.b_pt[b];
  DCHECK(i >= 0 && i < p.n_cams, "boundary camera", i, p.n_cams);
  DCHECK(j >= 0 && j < p.n_own_pts, "boundary point", j, p.n_own_pts);
  DCHECK(p.n_cam_side + b < p.n_records, "boundary record", p.n_cam_side + b, p.n_records);
  const double2 u = p.b_uv[b];
  const double4 lk = ld256(p.pts[p.roles[1]] + j), lb = ld256(p.lbar[p.roles[4]] + j);
  double cb[16], ck[16];
  load_cam16(p.cbarb[p.roles[4]] + (size_t)i * kCamStride, cb);
  load_cam16(p.cams[p.roles[1]] + (size_t)i * kCamStride, ck);
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  pt_terms<LOSS>(cb, lb.x, lb.y, lb.z, u, p, a[0], a[1], a[2], a[3]);
  pt_terms<LOSS>(ck, lk.x, lk.y, lk.z, u, p, a[4], a[5], a[6], a[7]);
  const int64_t r = p.n_cam_side + b;
  *rec_ptr(p, r, 0) = make_double4(a[0], a[1], a[2], a[3]);
  *rec_ptr(p, r, 1) = make_double4(a[4], a[5], a[6], a[7]);
}

__device__ void do_select(const IterParams& p);

// Rank-local sums of the camera partials (k_cam_solve blocks, 8 columns) and point partials (k_pt_sum blocks,
// 4 columns) in a fixed order by one block (any power-of-two size <= 256) -> p.local (a9).
// (noinline, arguments by value: its registers stay out of the kernels' allocation and no parameter copy)
struct FinalArgs {
  const double *cam_part, *pt_part, *inter_part;
  int32_t n_cam_eval_blocks, n_pt_blocks, n_inter_blocks;
  double* local;
};
__device__ __noinline__ void final_reduce(const FinalArgs p) {
  __shared__ double s[8][kGlobalCols];  // one row per warp (blockDim.x <= 256)
  const int nt = blockDim.x;
  double v[kGlobalCols];
  for (int c = 0; c < kGlobalCols; ++c) v[c] = 0.0;
  for (int b = threadIdx.x; b < p.n_cam_eval_blocks; b += nt) {
    const double* q = p.cam_part + (size_t)b * kCamEvalCols;
    v[0] += __ldcg(q + 0);
    v[1] += __ldcg(q + 1);
    v[3] += __ldcg(q + 2);
    v[5] += __ldcg(q + 3);
    v[6] += __ldcg(q + 4);
    v[7] += __ldcg(q + 5);
    v[8] += __ldcg(q + 6);
    v[9] += __ldcg(q + 7);
  }
  for (int b = threadIdx.x; b < p.n_pt_blocks; b += nt) {
    const double* q = p.pt_part + (size_t)b * kPtCols;
    v[2] += __ldcg(q + 0);
    v[4] += __ldcg(q + 1);
    v[5] += __ldcg(q + 2);
    v[6] += __ldcg(q + 3);
  }
  for (int b = threadIdx.x; b < p.n_inter_blocks; b += nt) {
    v[10] += __ldcg(p.inter_part + 2 * (size_t)b);
    v[11] += __ldcg(p.inter_part + 2 * (size_t)b + 1);
  }
  // warp shuffles, then the warps' rows in order (fixed order: deterministic); little shared memory, so the
  // kernels that end with it keep their occupancy and L1
#pragma unroll
  for (int c = 0; c < kGlobalCols; ++c)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[c] += __shfl_down_sync(0xffffffffu, v[c], off);
  if ((threadIdx.x & 31) == 0)
    for (int c = 0; c < kGlobalCols; ++c) s[threadIdx.x >> 5][c] = v[c];
  __syncthreads();
  if (threadIdx.x < kGlobalCols) {
    double t = 0.0;
    for (int w = 0; w < (nt + 31) / 32; ++w) t += s[w][threadIdx.x];
    p.local[threadIdx.x] = t;
  }
}

// Epilogue of every k_cam_solve and k_pt_sum block (the two kernels may run concurrently): after its partial is
// written, the block that finishes last (across both kernels) forms the rank-local sums and, without a
// communicator, takes the restart decision.
__device__ void finish_block(const IterParams& p) {
  __shared__ bool last;
  if (threadIdx.x < kCamEvalCols) __threadfence();  // the threads that wrote this block's partial
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(p.counter, 1) == p.n_cam_eval_blocks + p.n_pt_blocks - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  final_reduce(FinalArgs{p.cam_part, p.pt_part, p.inter_part, p.n_cam_eval_blocks, p.n_pt_blocks, p.n_inter_blocks,
                         p.local});
  if (threadIdx.x == 0) {
    *p.counter = 0;
    __threadfence();
    if (!p.has_comm || p.restart_scope == 1) do_select(p);  // a per-device decision needs no collective
  }
}

// Point solve (a7) over a grid-stride set of owned points: each point adds its observations' records in
// ascending (camera) order and takes the exact minimiser for both anchors.  The last block to finish forms the
// rank-local sums (a9) and, without a communicator, takes the restart decision (a9 + a10).  Deterministic.
// (measured at 2 CTAs/SM and 4 records per batch: 0.588 ms; 3 records 0.612, 6 records 0.652, 2 records at 3 or 4
// CTAs/SM 0.607 / 0.717, 4 records at 3 CTAs/SM spill: 1.14, a max-L1 carve-out 0.69)
__global__ void __launch_bounds__(kPtPassThreads, 2) k_pt_sum(IterParams p) {
  double qv[kPtCols] = {0, 0, 0, 0};
  for (int jj = blockIdx.x * kPtPassThreads + threadIdx.x; jj < p.n_own_pts; jj += gridDim.x * kPtPassThreads) {
    // highest point first: the camera pass writes the last cameras' records last, so theirs are the ones still in
    // L2, and (points numbered along the cameras) the highest points read them (8-rank shard of Final-13682:
    // 0.1078 -> 0.1060 ms; one rank unchanged)
    const int j = p.n_own_pts - 1 - jj;
    const double4 k4 = p.pts[p.roles[1]][j], b4 = p.lbar[p.roles[4]][j];
    const double lk[3] = {k4.x, k4.y, k4.z};
    const double lb[3] = {b4.x, b4.y, b4.z};
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int64_t o1 = p.p_ptr[j + 1];
    for (int64_t o = p.p_ptr[j]; o < o1; o += 4) {  // up to 4 records (8 x 32 B) in flight per thread
      int32_t r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) r[i] = o + i < o1 ? p.p_src[o + i] : -1;
#pragma unroll
      for (int i = 0; i < 4; ++i) DCHECK(r[i] < p.n_records && (r[i] >= 0 || o + i >= o1), "record", r[i], p.n_records);
      double4 A[4], B[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (r[i] >= 0) {
          A[i] = ld256_na(rec_ptr(p, r[i], 0));
          B[i] = ld256_na(rec_ptr(p, r[i], 1));
        }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (r[i] >= 0) {  // ascending observation order within the point
          acc[0] += A[i].x; acc[1] += A[i].y; acc[2] += A[i].z; acc[3] += A[i].w;
          acc[4] += B[i].x; acc[5] += B[i].y; acc[6] += B[i].z; acc[7] += B[i].w;
        }
    }
    double q[kPtCols];
    pt_finish(p, j, lb, lk, acc, q);
#pragma unroll
    for (int c = 0; c < kPtCols; ++c) qv[c] += q[c];
  }
  // block sums: warp shuffles, then one shared-memory step (deterministic order)
  __shared__ double ws[kPtPassThreads / 32][kPtCols];
#pragma unroll
  for (int c = 0; c < kPtCols; ++c) {
    double v = qv[c];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5][c] = v;
  }
  __syncthreads();
  if (threadIdx.x < kPtCols) {
    double v = 0;
    for (int w = 0; w < kPtPassThreads / 32; ++w) v += ws[w][threadIdx.x];
    p.pt_part[(size_t)blockIdx.x * kPtCols + threadIdx.x] = v;
  }
  finish_block(p);
}

// ------------------------------------------------------------------ a6: camera solve
// Sums of App. A of SURVEY.md (all in the anchor camera frame), derived from the 40 moments.
struct Sums {
  double Spp[9], Spb[9], Sbb[9], Slp[3], Slb[3], Sll, Spe[9], Seb[9], Sle[3];
};

__device__ __forceinline__ void derive_sums(const double* m, const double* d, Sums& S) {
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) S.Sbb[3 * a + b] = m[9 + a + b];
  double Sbbd[3];
  for (int a = 0; a < 3; ++a) Sbbd[a] = S.Sbb[3 * a] * d[0] + S.Sbb[3 * a + 1] * d[1] + S.Sbb[3 * a + 2] * d[2];
  S.Spp[0] = m[0];
  S.Spp[1] = S.Spp[3] = m[1];
  S.Spp[4] = m[2];
  S.Spp[2] = S.Spp[6] = d[0] * m[3] + d[1] * m[4] + d[2] * m[5];
  S.Spp[5] = S.Spp[7] = d[0] * m[6] + d[1] * m[7] + d[2] * m[8];
  S.Spp[8] = d[0] * Sbbd[0] + d[1] * Sbbd[1] + d[2] * Sbbd[2];
  for (int b = 0; b < 3; ++b) {
    S.Spb[b] = m[3 + b];
    S.Spb[3 + b] = m[6 + b];
    S.Spb[6 + b] = Sbbd[b];
  }
  S.Slb[0] = m[16];
  S.Slb[1] = m[17];
  S.Slb[2] = m[18];
  S.Slp[0] = m[14];
  S.Slp[1] = m[15];
  S.Slp[2] = d[0] * m[16] + d[1] * m[17] + d[2] * m[18];
  S.Sll = m[19];
  for (int a = 0; a < 3; ++a) {
    S.Spe[a] = m[20 + a];      // sum w ux e_a
    S.Spe[3 + a] = m[23 + a];  // sum w uy e_a
    S.Spe[6 + a] = d[0] * m[26 + a] + d[1] * m[29 + a] + d[2] * m[32 + a];  // sum w pz e_a
    for (int c = 0; c < 3; ++c) S.Seb[3 * a + c] = m[26 + 3 * c + a];       // sum w e_a b_c
    S.Sle[a] = m[35 + a];
  }
}

// Exact change of sum_j P_ij + xi/2 ||c - c_hat||^2 for a camera move (dR = R' - R_hat, dt, dd), from the sums
// (identity of SURVEY.md App. A; derivation in DESIGN.md "Trial decrease from moments").
__device__ double delta_P(const double* Rh, const Sums& S, const double* dR, const double* dt, const double* dd,
                          double xi) {
  double B[9];
  mat3_tmul(Rh, dR, B);  // R_hat^T dR = R_hat^T (A - I) R_hat
  const double c3[3] = {B[2], B[5], 1.0 + B[8]};
  double tau[3];
  for (int r = 0; r < 3; ++r) tau[r] = Rh[r] * dt[0] + Rh[3 + r] * dt[1] + Rh[6 + r] * dt[2];
  double BS[9];
  mat3_mul(B, S.Spp, BS);
  double T1 = 0;
  for (int k = 0; k < 9; ++k) T1 += BS[k] * B[k];
  double Sbbdd[3], Spbdd[3], Sebdd[3];
  for (int a = 0; a < 3; ++a) {
    Sbbdd[a] = S.Sbb[3 * a] * dd[0] + S.Sbb[3 * a + 1] * dd[1] + S.Sbb[3 * a + 2] * dd[2];
    Spbdd[a] = S.Spb[3 * a] * dd[0] + S.Spb[3 * a + 1] * dd[1] + S.Spb[3 * a + 2] * dd[2];
    Sebdd[a] = S.Seb[3 * a] * dd[0] + S.Seb[3 * a + 1] * dd[1] + S.Seb[3 * a + 2] * dd[2];
  }
  const double ddSbbdd = dd[0] * Sbbdd[0] + dd[1] * Sbbdd[1] + dd[2] * Sbbdd[2];
  const double c3n = c3[0] * c3[0] + c3[1] * c3[1] + c3[2] * c3[2];
  const double taun = tau[0] * tau[0] + tau[1] * tau[1] + tau[2] * tau[2];
  double BSpbdd[3], BSlp[3];
  for (int r = 0; r < 3; ++r) {
    BSpbdd[r] = B[3 * r] * Spbdd[0] + B[3 * r + 1] * Spbdd[1] + B[3 * r + 2] * Spbdd[2];
    BSlp[r] = B[3 * r] * S.Slp[0] + B[3 * r + 1] * S.Slp[1] + B[3 * r + 2] * S.Slp[2];
  }
  const double T2 = ddSbbdd * c3n;
  const double T3 = S.Sll * taun;
  const double T4 = 2.0 * (c3[0] * BSpbdd[0] + c3[1] * BSpbdd[1] + c3[2] * BSpbdd[2]);
  const double T5 = 2.0 * (tau[0] * BSlp[0] + tau[1] * BSlp[1] + tau[2] * BSlp[2]);
  const double T6 = 2.0 * (tau[0] * c3[0] + tau[1] * c3[1] + tau[2] * c3[2]) *
                    (S.Slb[0] * dd[0] + S.Slb[1] * dd[1] + S.Slb[2] * dd[2]);
  double T7 = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) T7 += B[3 * a + b] * S.Spe[3 * b + a];
  const double T8 = c3[0] * Sebdd[0] + c3[1] * Sebdd[1] + c3[2] * Sebdd[2];
  const double T9 = S.Sle[0] * tau[0] + S.Sle[1] * tau[1] + S.Sle[2] * tau[2];
  double prox = 0;
  for (int k = 0; k < 9; ++k) prox += dR[k] * dR[k];
  for (int k = 0; k < 3; ++k) prox += dt[k] * dt[k] + dd[k] * dd[k];
  return ((T1 + T2 + T3) + (T4 + T5 + T6)) + (T7 + T8 + T9) + 0.5 * xi * prox;
}

// Gauss-Newton normal equations of sum_j P_ij + xi/2 ||c - c_hat||^2 on the tangent (dtheta, dt, dd),
// left perturbation R = Exp(dtheta) R_hat.
__device__ void normal_equations(const double* Rh, const Sums& S, double xi, double* H, double* g) {
  for (int k = 0; k < 81; ++k) H[k] = 0.0;
  // theta-theta: 2 R (tr(Spp) I - Spp) R^T
  double Q[9];
  const double tr = S.Spp[0] + S.Spp[4] + S.Spp[8];
  for (int k = 0; k < 9; ++k) Q[k] = (k % 4 == 0 ? tr : 0.0) - S.Spp[k];
  double RQ[9], RQRt[9];
  mat3_mul(Rh, Q, RQ);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) RQRt[3 * r + c] = RQ[3 * r] * Rh[3 * c] + RQ[3 * r + 1] * Rh[3 * c + 1] + RQ[3 * r + 2] * Rh[3 * c + 2];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) H[9 * r + c] = 2.0 * RQRt[3 * r + c];
  // theta-t: 2 [R Slp]x ; t-theta its transpose
  double a[3];
  for (int r = 0; r < 3; ++r) a[r] = Rh[3 * r] * S.Slp[0] + Rh[3 * r + 1] * S.Slp[1] + Rh[3 * r + 2] * S.Slp[2];
  const double X[9] = {0, -a[2], a[1], a[2], 0, -a[0], -a[1], a[0], 0};
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      H[9 * r + 3 + c] = 2.0 * X[3 * r + c];
      H[9 * (3 + c) + r] = 2.0 * X[3 * r + c];
    }
  // theta-d: 2 R [sum w uy b^T ; -sum w ux b^T ; 0]
  const double N[9] = {S.Spb[3], S.Spb[4], S.Spb[5], -S.Spb[0], -S.Spb[1], -S.Spb[2], 0, 0, 0};
  double RN[9];
  mat3_mul(Rh, N, RN);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      H[9 * r + 6 + c] = 2.0 * RN[3 * r + c];
      H[9 * (6 + c) + r] = 2.0 * RN[3 * r + c];
    }
  // t-t: 2 Sll I;  t-d: 2 r3 Slb^T (r3 = R e3);  d-d: 2 Sbb
  for (int r = 0; r < 3; ++r) {
    H[9 * (3 + r) + 3 + r] = 2.0 * S.Sll;
    for (int c = 0; c < 3; ++c) {
      const double v = 2.0 * Rh[3 * r + 2] * S.Slb[c];
      H[9 * (3 + r) + 6 + c] = v;
      H[9 * (6 + c) + 3 + r] = v;
      H[9 * (6 + r) + 6 + c] = 2.0 * S.Sbb[3 * r + c];
    }
  }
  for (int k = 0; k < 9; ++k) H[9 * k + k] += xi * (k < 3 ? 2.0 : 1.0);
  // gradient: (R sum w p x e, R Sle, sum w e_z b)
  const double q[3] = {S.Spe[5] - S.Spe[7], S.Spe[6] - S.Spe[2], S.Spe[1] - S.Spe[3]};
  for (int r = 0; r < 3; ++r) {
    g[r] = Rh[3 * r] * q[0] + Rh[3 * r + 1] * q[1] + Rh[3 * r + 2] * q[2];
    g[3 + r] = Rh[3 * r] * S.Sle[0] + Rh[3 * r + 1] * S.Sle[1] + Rh[3 * r + 2] * S.Sle[2];
    g[6 + r] = S.Seb[6 + r];
  }
}

__host__ __device__ constexpr int tri(int r, int c) { return r * (r + 1) / 2 + c; }  // packed lower triangle

// a6 + a8, one thread per (camera, anchor); lanes 2i and 2i+1 hold camera i's accelerated (x-bar^k) and MM
// (x^k) subproblems.  Each thread sums its chunk partials (fixed order), builds the normal equations from the
// moments, takes one successful LM step, writes its candidate and the candidate's x-bar for the next iteration;
// the MM lane then evaluates the camera's part of E(x_acc|x^k) - F(x^k) and F(x^k) from its own (x^k) sums.
__global__ void __launch_bounds__(128) k_cam_solve(IterParams p) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = t < 2 * p.n_own_cams;
  const int i = valid ? (t >> 1) : 0, a = t & 1;  // a = 0: accelerated anchor x-bar^k, a = 1: x^k
  double m[kPartialStride];
  for (int k = 0; k < kPartialStride; ++k) m[k] = 0.0;
  double out[15], Rh[9], th[3], dh[3];
  Sums S;
  int accepted = -1;
  double dP_acc = 0.0;
  const double* ck = p.cams[p.roles[1]] + (size_t)i * kCamStride;
  if (valid) {
    DCHECK(p.cam_chunk_ptr[i] <= p.cam_chunk_ptr[i + 1] && p.cam_chunk_ptr[i + 1] <= p.n_chunks, "camera chunks",
           p.cam_chunk_ptr[i + 1], p.n_chunks);
    for (int c = p.cam_chunk_ptr[i]; c < p.cam_chunk_ptr[i + 1]; ++c) {
      const double* src = p.partial + ((size_t)c * 2 + a) * kPartialStride;
      for (int k = 0; k < kPartialStride; ++k) m[k] += src[k];
    }
    const double* anchor = (a == 0 ? p.cbarb[p.roles[4]] : p.cams[p.roles[1]]) + (size_t)i * kCamStride;
    for (int k = 0; k < 9; ++k) Rh[k] = anchor[k];
    for (int k = 0; k < 3; ++k) th[k] = anchor[9 + k];
    for (int k = 0; k < 3; ++k) dh[k] = anchor[12 + k];
    // the camera pass accumulated the error moments (slots 20..37: e times u_x, u_y, 1, s, s^2, lambda) in the
    // world frame: rotate each 3-vector into the anchor camera frame, e = R_hat^T (R e)
    for (int gq = 0; gq < 6; ++gq) {
      double* v = m + 20 + 3 * gq;
      const double a0 = v[0], a1 = v[1], a2 = v[2];
      v[0] = fma(Rh[0], a0, fma(Rh[3], a1, Rh[6] * a2));
      v[1] = fma(Rh[1], a0, fma(Rh[4], a1, Rh[7] * a2));
      v[2] = fma(Rh[2], a0, fma(Rh[5], a1, Rh[8] * a2));
    }
    derive_sums(m, dh, S);
    double H[81], g[9];
    normal_equations(Rh, S, p.xi, H, g);
    double sc[9];
    for (int k = 0; k < 9; ++k) sc[k] = 1.0 / sqrt(H[9 * k + k]);
    for (int r = 0; r < 9; ++r) {
      g[r] *= sc[r];
      for (int c = 0; c < 9; ++c) H[9 * r + c] *= sc[r] * sc[c];
    }
    for (int k = 0; k < 15; ++k) out[k] = anchor[k];
    double mu = p.mu0;
#pragma unroll 1
    for (int tau = 0; tau < p.max_trials; ++tau, mu *= p.mu_up) {
      // Cholesky of (H + mu diag H) in the Jacobi-scaled variables; fully unrolled (packed lower triangle in
      // registers).  A non-positive pivot makes the trial fail (Q3).
      double L[45];
      bool ok = true;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        double s = H[9 * j + j] * (1.0 + mu);
#pragma unroll
        for (int k = 0; k < j; ++k) s -= L[tri(j, k)] * L[tri(j, k)];
        ok = ok && (s > 0);
        const double ljj = sqrt(s > 0 ? s : 1.0);
        L[tri(j, j)] = ljj;
        const double il = 1.0 / ljj;
#pragma unroll
        for (int r = j + 1; r < 9; ++r) {
          double v = H[9 * r + j];
#pragma unroll
          for (int k = 0; k < j; ++k) v -= L[tri(r, k)] * L[tri(j, k)];
          L[tri(r, j)] = v * il;
        }
      }
      if (!ok) continue;
      double y[9], x[9];
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        double v = -g[r];
#pragma unroll
        for (int k = 0; k < r; ++k) v -= L[tri(r, k)] * y[k];
        y[r] = v / L[tri(r, r)];
      }
#pragma unroll
      for (int r = 8; r >= 0; --r) {
        double v = y[r];
#pragma unroll
        for (int k = r + 1; k < 9; ++k) v -= L[tri(k, r)] * x[k];
        x[r] = v / L[tri(r, r)];
      }
      double delta[9];
      for (int k = 0; k < 9; ++k) delta[k] = x[k] * sc[k];
      double EmI[9], dR[9];
      expm_minus_identity(delta, EmI);
      mat3_mul(EmI, Rh, dR);  // (Exp(dtheta) - I) R_hat
      const double dP = delta_P(Rh, S, dR, delta + 3, delta + 6, p.xi);
      if (dP < 0.0) {  // strict decrease: accept ("one successful inner LM step")
        for (int k = 0; k < 9; ++k) out[k] = Rh[k] + dR[k];
        for (int k = 0; k < 3; ++k) out[9 + k] = th[k] + delta[3 + k];
        for (int k = 0; k < 3; ++k) out[12 + k] = dh[k] + delta[6 + k];
        accepted = tau;
        dP_acc = dP;
        break;
      }
    }
  }
  if (valid) {
    double* dst = p.cams[p.roles[2 + a]] + (size_t)i * kCamStride;
    for (int k = 0; k < 15; ++k) dst[k] = out[k];
    dst[15] = 0.0;
    p.decisions[2 * i + a] = accepted;
    // x-bar^{k+1} of this candidate (used if the restart test selects it): eqs. nesterov_x with gamma^{(k+1)}
    double cb[16];
    extrapolate_camera(out, ck, sched_gamma_next(p.sched[0], p.accelerate), cb);
    double* cdst = p.cbarb[p.roles[5 + a]] + (size_t)i * kCamStride;
    for (int k = 0; k < 16; ++k) cdst[k] = cb[k];
    if (p.sendbuf)  // boundary camera: this anchor's candidate and its x-bar straight into its halo send slots
      for (int s = p.cam_send_ptr[i]; s < p.cam_send_ptr[i + 1]; ++s) {
        double* b = p.sendbuf + p.cam_send_off[s];
        for (int k = 0; k < 15; ++k) b[15 * a + k] = out[k];
        for (int k = 0; k < 16; ++k) b[30 + 16 * a + k] = cb[k];
      }
  }
  // camera part of E(x_acc|x^k) on the MM lane: the accelerated candidate comes from the partner lane
  double ca[15];
  for (int k = 0; k < 15; ++k) ca[k] = __shfl_xor_sync(0xffffffffu, out[k], 1);
  const int acc_accepted = __shfl_xor_sync(0xffffffffu, accepted, 1);
  double q[kCamEvalCols];
  for (int k = 0; k < kCamEvalCols; ++k) q[k] = 0.0;
  if (valid && a == 1) {
    double dR[9], dt[3], dd[3];
    for (int k = 0; k < 9; ++k) dR[k] = ca[k] - Rh[k];
    for (int k = 0; k < 3; ++k) {
      dt[k] = ca[9 + k] - th[k];
      dd[k] = ca[12 + k] - dh[k];
    }
    q[0] = m[39];  // F_i = sum rho / 2 (slot 38 unused)
    q[1] = delta_P(Rh, S, dR, dt, dd, p.xi);
    q[2] = dP_acc;
    double sa = 0, sm = 0;
    for (int k = 0; k < 15; ++k) {
      sa += (ca[k] - ck[k]) * (ca[k] - ck[k]);
      sm += (out[k] - ck[k]) * (out[k] - ck[k]);
    }
    q[3] = sa;
    q[4] = sm;
    q[5] = m[40];
    q[6] = acc_accepted < 0 ? 1.0 : 0.0;
    q[7] = accepted < 0 ? 1.0 : 0.0;
  }
  __shared__ double sq[kCamEvalCols][128];
  for (int c = 0; c < kCamEvalCols; ++c) sq[c][threadIdx.x] = q[c];
  __syncthreads();
  for (int st = 64; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int c = 0; c < kCamEvalCols; ++c) sq[c][threadIdx.x] += sq[c][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x < kCamEvalCols) p.cam_part[(size_t)blockIdx.x * kCamEvalCols + threadIdx.x] = sq[threadIdx.x][0];
  finish_block(p);
}

// ------------------------------------------------------------------ a9 + a10: restart test and selection
// The global test alone (D2), on the allreduced sums — the same arithmetic as do_select.
__device__ __forceinline__ bool restart_decision(const IterParams& p) {
  const double* G = p.global;
  const double F = G[0];
  const double Fbar = (1.0 - p.eta) * p.sched[1] + p.eta * F;
  const double Eacc = F + (G[1] + G[2]);
  return p.accelerate ? (Eacc > Fbar) : true;
}

__device__ void do_select(const IterParams& p) {
  double s_next;
  const double gamma = sched_gamma(p.sched[0], p.accelerate, &s_next);
  const bool dev = p.restart_scope == 1;
  // Global test (D2): the allreduced sums.  Per device (eqs. Fak, lFak, Eak; reading DN1): this rank's sums,
  //   F^{a(k)} = F_kappa(x^k) + D^{a(k)},  D^{a(k)} = D^{a(k-1)} + (1/2) sum_inter sign (dP_ij - dQ_ij),
  // F_kappa = the rank's camera-side F with inter-device pairs at weight 1/2 (local[0] + local[10]).
  const double* G = dev ? p.local : p.global;
  const double D = dev ? p.sched[3] + G[11] : 0.0;
  const double F = dev ? (G[0] + G[10]) + D : G[0];
  const double Fbar = (1.0 - p.eta) * p.sched[1] + p.eta * F;  // eq. lFak
  const double Eacc = F + (G[1] + G[2]);                        // eq. Eak: E(x_acc | x^k)
  const double Emm = F + (G[3] + G[4]);
  // Alg. 1, strict ">"; the global test through restart_decision so that k_unpack's copy agrees bitwise
  const bool restart = dev ? (p.accelerate ? (Eacc > Fbar) : true) : restart_decision(p);
  const int64_t k = (int64_t)p.sched[2];
  double* tr = p.trace + (size_t)(k % p.trace_cap) * kTraceCols;
  tr[0] = dev ? G[0] + G[10] : F;  // per device with a communicator: replaced by the global F in k_trace_post
  tr[1] = Fbar;
  tr[2] = Eacc;
  tr[3] = (p.accelerate && restart) ? 1.0 : 0.0;
  tr[4] = Emm;
  tr[5] = restart ? G[6] : G[5];
  tr[6] = gamma;
  tr[7] = G[7];
  tr[8] = G[8];
  tr[9] = G[9];
  tr[10] = F;
  if (dev) p.sched[3] = D;
  const int r0 = p.roles[0], r1 = p.roles[1], r2 = p.roles[2], r3 = p.roles[3];
  p.roles[0] = r1;                 // x^{k}   -> x^{k-1}
  p.roles[1] = restart ? r3 : r2;  // x^{k+1} = x_mm (restart, Alg. 1) or x_acc (L414)
  p.roles[2] = r0;
  p.roles[3] = restart ? r2 : r3;
  const int b4 = p.roles[4], b5 = p.roles[5], b6 = p.roles[6];
  p.roles[4] = restart ? b6 : b5;  // x-bar^{k+1} of the selected candidate
  p.roles[5] = b4;                 // the other two buffers take the next candidates' x-bar
  p.roles[6] = restart ? b5 : b6;
  p.sched[0] = s_next;
  p.sched[1] = Fbar;
  p.sched[2] = (double)(k + 1);
}

__global__ void k_select(IterParams p) {
  if (threadIdx.x == 0 && blockIdx.x == 0) do_select(p);
}

// Per-device restart with a communicator: the decision was local; the allreduce then supplies the global
// columns of the trace row just written (F, degenerate pairs, cameras without an accepted trial).
__global__ void k_trace_post(IterParams p) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t k = (int64_t)p.sched[2] - 1;
  double* tr = p.trace + (size_t)(k % p.trace_cap) * kTraceCols;
  tr[0] = p.global[0];
  tr[7] = p.global[7];
  tr[8] = p.global[8];
  tr[9] = p.global[9];
}

// Inter-device pair terms of the per-device metrics (eq. DEalpha at x = x^k, anchor x^{k-1}; DN1).
// For a pair with sign s (+1: this rank owns the camera, -1: it owns the point):
//   col 0: -s F_ij(x^k) / 2           (F_kappa counts an inter-device pair at weight 1/2 on each side)
//   col 1:  s (dP_ij - dQ_ij) / 2      (dP_ij = P_ij(c^k|x^{k-1}) - P_ij(c^{k-1}|x^{k-1}), dQ_ij likewise: the
//                                        anchor-relative forms w dr.(dr + R e), w (lam dl).(lam dl - R e))
template <int LOSS>
__global__ void __launch_bounds__(kInterThreads) k_inter(IterParams p) {
  double v0 = 0.0, v1 = 0.0;
  const int64_t b = blockIdx.x * (int64_t)kInterThreads + threadIdx.x;
  if (b < p.n_inter) {
    const int32_t i = p.i_cam[b], j = p.i_pt[b];
    DCHECK(i >= 0 && i < p.n_cams, "inter camera", i, p.n_cams);
    DCHECK(j >= 0 && j < p.n_pts, "inter point", j, p.n_pts);
    const double sg = (double)p.i_sign[b];
    const double2 u = p.i_uv[b];
    const double* ck = p.cams[p.roles[1]] + (size_t)i * kCamStride;
    const double* cp = p.cams[p.roles[0]] + (size_t)i * kCamStride;
    const double4 lk = p.pts[p.roles[1]][j], lp = p.pts[p.roles[0]][j];
    const double s = fma(u.x, u.x, u.y * u.y);
    // anchor x^{k-1}: ray, lambda, R e, w (eqs. ray, gamma, error, w)
    const double pzp = fma(s, fma(s, cp[14], cp[13]), cp[12]);
    const double rpx = fma(cp[0], u.x, fma(cp[1], u.y, cp[2] * pzp));
    const double rpy = fma(cp[3], u.x, fma(cp[4], u.y, cp[5] * pzp));
    const double rpz = fma(cp[6], u.x, fma(cp[7], u.y, cp[8] * pzp));
    const double vx = lp.x - cp[9], vy = lp.y - cp[10], vz = lp.z - cp[11];
    const double nv = fma(vx, vx, fma(vy, vy, vz * vz));
    if (nv > p.eps2) {
      const double lam = fma(vx, rpx, fma(vy, rpy, vz * rpz)) / nv;
      const double ex = fma(-lam, vx, rpx), ey = fma(-lam, vy, rpy), ez = fma(-lam, vz, rpz);
      const double w = loss_eval<LOSS, false>(fma(ex, ex, fma(ey, ey, ez * ez)), p.delta, p.delta2, p.idelta2,
                                               nullptr);
      // camera move: dr = R^k p(d^k) - R^{k-1} p(d^{k-1}) + lam (t^k - t^{k-1})
      const double pzk = fma(s, fma(s, ck[14], ck[13]), ck[12]);
      const double dx = fma(ck[0], u.x, fma(ck[1], u.y, ck[2] * pzk)) - rpx + lam * (ck[9] - cp[9]);
      const double dy = fma(ck[3], u.x, fma(ck[4], u.y, ck[5] * pzk)) - rpy + lam * (ck[10] - cp[10]);
      const double dz = fma(ck[6], u.x, fma(ck[7], u.y, ck[8] * pzk)) - rpz + lam * (ck[11] - cp[11]);
      const double dP = w * fma(dx, dx + ex, fma(dy, dy + ey, dz * (dz + ez)));
      const double mx = lam * (lk.x - lp.x), my = lam * (lk.y - lp.y), mz = lam * (lk.z - lp.z);
      const double dQ = w * fma(mx, mx - ex, fma(my, my - ey, mz * (mz - ez)));
      v1 = 0.5 * sg * (dP - dQ);
    }
    // F_ij(x^k) (eq. Fij)
    const double pz = fma(s, fma(s, ck[14], ck[13]), ck[12]);
    const double rx = fma(ck[0], u.x, fma(ck[1], u.y, ck[2] * pz));
    const double ry = fma(ck[3], u.x, fma(ck[4], u.y, ck[5] * pz));
    const double rz = fma(ck[6], u.x, fma(ck[7], u.y, ck[8] * pz));
    const double wx = lk.x - ck[9], wy = lk.y - ck[10], wz = lk.z - ck[11];
    const double nw = fma(wx, wx, fma(wy, wy, wz * wz));
    if (nw > p.eps2) {
      const double lam = fma(wx, rx, fma(wy, ry, wz * rz)) / nw;
      const double ex = fma(-lam, wx, rx), ey = fma(-lam, wy, ry), ez = fma(-lam, wz, rz);
      double rho;
      loss_eval<LOSS, true>(fma(ex, ex, fma(ey, ey, ez * ez)), p.delta, p.delta2, p.idelta2, &rho);
      v0 = -0.25 * sg * rho;  // -s F_ij / 2, F_ij = rho / 2
    }
  }
  __shared__ double s0[kInterThreads], s1[kInterThreads];
  s0[threadIdx.x] = v0;
  s1[threadIdx.x] = v1;
  __syncthreads();
  for (int st = kInterThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      s0[threadIdx.x] += s0[threadIdx.x + st];
      s1[threadIdx.x] += s1[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.inter_part[2 * (size_t)blockIdx.x] = s0[0];
    p.inter_part[2 * (size_t)blockIdx.x + 1] = s1[0];
  }
}

// Create time: sum the k_inter partials into local[10], local[11] (fixed order).
__global__ void k_reduce_inter(IterParams p) {
  __shared__ double s0[256], s1[256];
  double a = 0, b = 0;
  for (int q = threadIdx.x; q < p.n_inter_blocks; q += 256) {
    a += p.inter_part[2 * (size_t)q];
    b += p.inter_part[2 * (size_t)q + 1];
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = b;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      s0[threadIdx.x] += s0[threadIdx.x + st];
      s1[threadIdx.x] += s1[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.local[10] = s0[0];
    p.local[11] = s1[0];
  }
}

// x-bar^k of every local camera and point from x^k, x^{k-1} (create / set_state); writes the role-selected
// x-bar buffers
__global__ void k_lbar_all(IterParams p) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const double gamma = sched_gamma(p.sched[0], p.accelerate, nullptr);
  if (j < p.n_pts) {
    const double4 k4 = p.pts[p.roles[1]][j], p4 = p.pts[p.roles[0]][j];
    p.lbar[p.roles[4]][j] = make_double4(fma(gamma, k4.x - p4.x, k4.x), fma(gamma, k4.y - p4.y, k4.y),
                                         fma(gamma, k4.z - p4.z, k4.z), 0.0);
  }
  if (j < p.n_cams)
    extrapolate_camera(p.cams[p.roles[1]] + (size_t)j * kCamStride, p.cams[p.roles[0]] + (size_t)j * kCamStride, gamma,
                       p.cbarb[p.roles[4]] + (size_t)j * kCamStride);
}

// ------------------------------------------------------------------ halo pack / unpack (x^k)
// Both candidates of each boundary variable (before the restart decision): camera [acc 15 | mm 15],
// point [acc 3 | mm 3].
__global__ void k_pack(IterParams p, const int32_t* cam_idx, const int64_t* cam_off, int32_t n_cam,
                       const int32_t* pt_idx, const int64_t* pt_off, int32_t n_pt, double* buf, int selected) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // before the decision: [acc | mm] candidates; after a local decision (selected): [x^{k+1} | x^{k+1}].
  // Cameras: one warp per camera, one double per lane; points: one thread per point.
  const int ra = selected ? p.roles[1] : p.roles[2], rm = selected ? p.roles[1] : p.roles[3];
  const int n_cam_threads = 64 * n_cam;
  if (t < n_cam_threads) {  // two warps per camera: lanes 0..61 copy one double each
    const int e = t >> 6, c = t & 63;
    DCHECK(cam_idx[e] >= 0 && cam_idx[e] < p.n_own_cams, "send camera", cam_idx[e], p.n_own_cams);
    const size_t i = (size_t)cam_idx[e] * kCamStride;
    double v = 0.0;
    if (c < 15)
      v = p.cams[ra][i + c];
    else if (c < 30)
      v = p.cams[rm][i + c - 15];
    else if (c < 46)  // x-bar of either outcome (before the decision) or of the selected one (after)
      v = p.cbarb[selected ? p.roles[4] : p.roles[5]][i + c - 30];
    else if (c < 62)
      v = p.cbarb[selected ? p.roles[4] : p.roles[6]][i + c - 46];
    if (c < kHaloCam) buf[cam_off[e] + c] = v;
  } else if (t < n_cam_threads + n_pt) {
    const int q = t - n_cam_threads;
    DCHECK(pt_idx[q] >= 0 && pt_idx[q] < p.n_own_pts, "send point", pt_idx[q], p.n_own_pts);
    const double4 la = p.pts[ra][pt_idx[q]], lm = p.pts[rm][pt_idx[q]];
    double* b = buf + pt_off[q];
    b[0] = la.x;
    b[1] = la.y;
    b[2] = la.z;
    b[3] = lm.x;
    b[4] = lm.y;
    b[5] = lm.z;
  }
}

// After the restart decision (roles rotated, roles[4] = 1 iff the MM candidate was kept): the selected candidate
// becomes the halo entry of x^{k+1}, and its x-bar^{k+1} is formed from the cached x^k (eqs. nesterov_x).
__global__ void k_unpack(IterParams p, const int32_t* cam_idx, const int64_t* cam_off, int32_t n_cam,
                         const int32_t* pt_idx, const int64_t* pt_off, int32_t n_pt, const double* buf,
                         int select_inside) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // after the decision: x^{k+1} = roles[1], x^k = roles[0], x-bar buffer roles[4], gamma^{(k+1)} from s^{(k+1)};
  // with select_inside the decision is still to be committed: every thread derives the same outcome
  // (sel: which half of the received record; without select_inside both halves carry x^{k+1})
  int sel, r_new, r_old, xbuf;
  double gamma;
  if (select_inside) {
    const bool restart = restart_decision(p);
    sel = restart ? 1 : 0;
    r_new = restart ? p.roles[3] : p.roles[2];
    r_old = p.roles[1];
    xbuf = p.roles[5 + sel];
    gamma = sched_gamma_next(p.sched[0], p.accelerate);
  } else {
    sel = 0;
    r_new = p.roles[1];
    r_old = p.roles[0];
    xbuf = p.roles[4];
    gamma = sched_gamma(p.sched[0], p.accelerate, nullptr);
  }
  const int64_t n_cam_thr = (int64_t)n_cam * 32;  // one warp per halo camera: lane k < 15 copies x_k, 16 + k x-bar_k
  if (t < n_cam_thr) {  // x^{k+1} and its x-bar^{k+1} as the owner computed them (coalesced 31-double records)
    const int e = t >> 5, lane = t & 31;
    DCHECK(cam_idx[e] >= p.n_own_cams && cam_idx[e] < p.n_cams, "halo camera", cam_idx[e], p.n_cams);
    const size_t i = (size_t)cam_idx[e] * kCamStride;
    const double* src = buf + cam_off[e];
    if (lane < 16) p.cams[r_new][i + lane] = lane < 15 ? src[15 * sel + lane] : 0.0;
    else p.cbarb[xbuf][i + lane - 16] = src[30 + 16 * sel + lane - 16];
  } else if (t < n_cam_thr + n_pt) {
    const int q = (int)(t - n_cam_thr);
    DCHECK(pt_idx[q] >= p.n_own_pts && pt_idx[q] < p.n_pts, "halo point", pt_idx[q], p.n_pts);
    const double* b = buf + pt_off[q] + 3 * sel;
    const double4 lp = p.pts[r_old][pt_idx[q]];
    p.pts[r_new][pt_idx[q]] = make_double4(b[0], b[1], b[2], 0.0);
    p.lbar[xbuf][pt_idx[q]] = make_double4(fma(gamma, b[0] - lp.x, b[0]), fma(gamma, b[1] - lp.y, b[1]),
                                          fma(gamma, b[2] - lp.z, b[2]), 0.0);
  }
  if (select_inside) {  // the last block commits the decision (roles, schedule, trace) once every block is done
    __shared__ bool last;
    __syncthreads();  // (do_select reads only the allreduced sums and the roles every block has read by now)
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(p.counter, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      *p.counter = 0;
      __threadfence();
      do_select(p);
    }
  }
}

// ------------------------------------------------------------------ launchers
static inline int blocks(int64_t n, int t) { return (int)((n + t - 1) / t); }

int launch_lbar_all(const IterParams& p, cudaStream_t st) {
  const int64_t n = p.n_pts > p.n_cams ? p.n_pts : p.n_cams;
  if (n == 0) return 0;
  k_lbar_all<<<blocks(n, 256), 256, 0, st>>>(p);
  return 1;
}

template <int LOSS>
static void cam_launch(const IterParams& p, cudaStream_t st) {
  constexpr size_t sm = sizeof(double) * kCamSmemDoubles;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_cam_pass<LOSS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_cam_pass<LOSS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  if (p.cam_shared_ctas)
    k_cam_pass<LOSS, true><<<p.n_chunks, kCamPassThreads, sm, st>>>(p);
  else
    k_cam_pass<LOSS, false><<<2 * p.n_chunks, kCamPassThreads, sm, st>>>(p);
}

int launch_cam_pass(const IterParams& p, cudaStream_t st) {
  if (p.n_chunks == 0) return 0;
  switch (p.loss) {
    case kHuber: cam_launch<kHuber>(p, st); break;
    case kCauchy: cam_launch<kCauchy>(p, st); break;
    default: cam_launch<kTrivial>(p, st); break;
  }
  return 1;
}

int launch_pt_pass(const IterParams& p, cudaStream_t st) {
  int n = 0;
  if (p.n_boundary > 0) {
    const int nb = blocks(p.n_boundary, 256);
    switch (p.loss) {
      case kHuber: k_pt_boundary<kHuber><<<nb, 256, 0, st>>>(p); break;
      case kCauchy: k_pt_boundary<kCauchy><<<nb, 256, 0, st>>>(p); break;
      default: k_pt_boundary<kTrivial><<<nb, 256, 0, st>>>(p); break;
    }
    ++n;
  }
  return n;
}

int launch_pt_sum(const IterParams& p, cudaStream_t st) {
  k_pt_sum<<<p.n_pt_blocks, kPtPassThreads, 0, st>>>(p);
  return 1;
}

int launch_cam_solve(const IterParams& p, cudaStream_t st) {
  if (p.n_own_cams == 0) return 0;
  k_cam_solve<<<blocks(2 * (int64_t)p.n_own_cams, 128), 128, 0, st>>>(p);
  return 1;
}


int launch_select(const IterParams& p, cudaStream_t st) {
  k_select<<<1, 32, 0, st>>>(p);
  return 1;
}

int launch_objective(const IterParams& p, cudaStream_t st) {
  int n = 0;
  if (p.n_chunks > 0) {
    switch (p.loss) {
      case kHuber: k_objective<kHuber><<<p.n_chunks, kCamPassThreads, 0, st>>>(p); break;
      case kCauchy: k_objective<kCauchy><<<p.n_chunks, kCamPassThreads, 0, st>>>(p); break;
      default: k_objective<kTrivial><<<p.n_chunks, kCamPassThreads, 0, st>>>(p); break;
    }
    ++n;
  }
  k_reduce_objective<<<1, 256, 0, st>>>(p);
  return n + 1;
}

int launch_pixel_error(const IterParams& p, int role, double* out, double* resid, cudaStream_t st) {
  int n = 0;
  if (p.n_chunks > 0) {
    k_pixel_error<<<p.n_chunks, kCamPassThreads, 0, st>>>(p, role, resid);
    ++n;
  }
  k_reduce_pixel_error<<<1, 256, 0, st>>>(p, out);
  return n + 1;
}

int launch_pack(const IterParams& p, const int32_t* cam_idx, const int64_t* cam_off, int32_t n_cam,
                const int32_t* pt_idx, const int64_t* pt_off, int32_t n_pt, double* buf, int selected,
                cudaStream_t st) {
  if (n_cam + n_pt == 0) return 0;
  k_pack<<<blocks(64 * (int64_t)n_cam + n_pt, 256), 256, 0, st>>>(p, cam_idx, cam_off, n_cam, pt_idx, pt_off, n_pt,
                                                                  buf, selected);
  return 1;
}

int launch_inter(const IterParams& p, cudaStream_t st) {
  if (p.n_inter_blocks == 0) return 0;
  switch (p.loss) {
    case kHuber: k_inter<kHuber><<<p.n_inter_blocks, kInterThreads, 0, st>>>(p); break;
    case kCauchy: k_inter<kCauchy><<<p.n_inter_blocks, kInterThreads, 0, st>>>(p); break;
    default: k_inter<kTrivial><<<p.n_inter_blocks, kInterThreads, 0, st>>>(p); break;
  }
  return 1;
}

int launch_reduce_inter(const IterParams& p, cudaStream_t st) {
  k_reduce_inter<<<1, 256, 0, st>>>(p);
  return 1;
}

int launch_trace_post(const IterParams& p, cudaStream_t st) {
  k_trace_post<<<1, 32, 0, st>>>(p);
  return 1;
}

int launch_unpack(const IterParams& p, const int32_t* cam_idx, const int64_t* cam_off, int32_t n_cam,
                  const int32_t* pt_idx, const int64_t* pt_off, int32_t n_pt, const double* buf, int select_inside,
                  cudaStream_t st) {
  if (n_cam + n_pt == 0) return 0;
  k_unpack<<<blocks((int64_t)n_cam * 32 + n_pt, 256), 256, 0, st>>>(p, cam_idx, cam_off, n_cam, pt_idx, pt_off, n_pt, buf,
                                                      select_inside);
  return 1;
}

// ------------------------------------------------------------------ state readback
// owned points (double4, w unused) -> packed xyz, so that one D2H lands in the caller's N x 3 array
__global__ void k_pts_xyz(const double4* __restrict__ src, double* __restrict__ dst, int32_t n) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double4 v = src[j];
  dst[3 * (int64_t)j] = v.x;
  dst[3 * (int64_t)j + 1] = v.y;
  dst[3 * (int64_t)j + 2] = v.z;
}
__global__ void k_xyz_pts(const double* __restrict__ src, double4* __restrict__ dst, int32_t n) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  dst[j] = make_double4(src[3 * (int64_t)j], src[3 * (int64_t)j + 1], src[3 * (int64_t)j + 2], 0.0);
}
int launch_xyz_pts(const double* src, double4* dst, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_xyz_pts<<<blocks(n, 256), 256, 0, st>>>(src, dst, n);
  return 1;
}
int launch_pts_xyz(const double4* src, double* dst, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_pts_xyz<<<blocks(n, 256), 256, 0, st>>>(src, dst, n);
  return 1;
}

// ------------------------------------------------------------------ create-time point side on the device
// (one rank, input sorted by (camera, point): the observation index is the camera-side record index)
__global__ void k_iota(int32_t* v, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}
__global__ void k_fill_i32(int32_t* v, int64_t n, int32_t x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = x;
}
__global__ void k_min_camera(const int32_t* cam, const int32_t* pt, int64_t K, int32_t* key) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < K) atomicMin(key + pt[q], cam[q]);
}
// consecutive points whose smallest cameras lie more than `far` ids apart (shard.h order_owned_points)
__global__ void k_count_jumps(const int32_t* key, int64_t n, int32_t far, unsigned long long* out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool jump = j + 1 < n && abs(key[j + 1] - key[j]) > far;
  const unsigned m = __ballot_sync(0xffffffffu, jump);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, (unsigned long long)__popc(m));
}
// CSR offsets from keys sorted ascending: ptr[j] = first position with key >= j, ptr[N] = K
__global__ void k_ptr_from_sorted(const int32_t* keys, int64_t K, int32_t N, int64_t* ptr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int32_t k = keys[i], kp = i > 0 ? keys[i - 1] : -1;
  for (int32_t j = kp + 1; j <= k; ++j) ptr[j] = i;
  if (i == K - 1)
    for (int32_t j = k + 1; j <= N; ++j) ptr[j] = K;
}

static inline unsigned grid(int64_t n) { return (unsigned)((n + 255) / 256); }

// Carve aligned pieces out of a scratch region.
static void* carve(char*& p, size_t bytes) {
  void* r = p;
  p += (bytes + 255) & ~size_t(255);
  return r;
}

int64_t count_point_jumps_device(const int32_t* d_cam, const int32_t* d_pt, int64_t K, int32_t N, int32_t far,
                                 void* scratch, cudaStream_t st) {
  char* sp = static_cast<char*>(scratch);
  int32_t* key = static_cast<int32_t*>(carve(sp, sizeof(int32_t) * (size_t)(N > 0 ? N : 1)));
  unsigned long long* cnt = static_cast<unsigned long long*>(carve(sp, sizeof(unsigned long long)));
  cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st);
  if (N > 0) k_fill_i32<<<grid(N), 256, 0, st>>>(key, N, 0x7fffffff);
  if (K > 0) k_min_camera<<<grid(K), 256, 0, st>>>(d_cam, d_pt, K, key);
  if (N > 1) k_count_jumps<<<grid(N), 256, 0, st>>>(key, N, far, cnt);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, st);
  return cudaStreamSynchronize(st) == cudaSuccess ? (int64_t)h : -1;
}

int sort_point_side_device(const int32_t* d_pt, int64_t K, int32_t N, int32_t* d_src, int64_t* d_ptr, void* scratch,
                           size_t scratch_bytes, cudaStream_t st) {
  if (K == 0) {
    cudaMemsetAsync(d_ptr, 0, sizeof(int64_t) * ((size_t)N + 1), st);
    return cudaStreamSynchronize(st) == cudaSuccess ? 0 : -1;
  }
  int bits = 1;
  while ((int64_t(1) << bits) < (int64_t)N) ++bits;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_pt, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)K, 0, bits, st);
  char* sp = static_cast<char*>(scratch);
  int32_t* vals = static_cast<int32_t*>(carve(sp, sizeof(int32_t) * (size_t)K));
  int32_t* keys_out = static_cast<int32_t*>(carve(sp, sizeof(int32_t) * (size_t)K));
  void* tmp = carve(sp, tmp_bytes);
  if ((size_t)(sp - static_cast<char*>(scratch)) > scratch_bytes) return -1;
  k_iota<<<grid(K), 256, 0, st>>>(vals, K);
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, d_pt, keys_out, vals, d_src, (int)K, 0, bits, st);  // stable
  k_ptr_from_sorted<<<grid(K), 256, 0, st>>>(keys_out, K, N, d_ptr);
  return cudaStreamSynchronize(st) == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : -1;
}


// Create time, one rank: the observations' indices checked on the device (the arrays go there anyway), whether
// they are sorted by (camera, point) strictly (so also free of duplicate pairs), and — when they are — each
// camera's first observation.  bad_min: smallest k with an index out of range (K if none).
__global__ void k_validate_sorted(const int32_t* cam, const int32_t* pt, int64_t K, int64_t M, int64_t N,
                                  unsigned long long* bad_min, int* unsorted, int64_t* cptr) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int32_t c = cam[k], j = pt[k];
  if (c < 0 || c >= M || j < 0 || j >= N) {
    atomicMin(bad_min, (unsigned long long)k);
    return;
  }
  int32_t prev = -1;
  if (k > 0) {
    prev = cam[k - 1];
    const int32_t jp = pt[k - 1];
    if (!(prev < c || (prev == c && jp < j))) atomicOr(unsorted, 1);
  }
  for (int64_t i = prev + 1 > 0 ? prev + 1 : 0; i <= c; ++i) cptr[i] = k;  // cameras starting at k
  if (k == K - 1)
    for (int64_t i = (int64_t)c + 1; i <= M; ++i) cptr[i] = K;
}

int validate_sorted_device(const int32_t* d_cam, const int32_t* d_pt, int64_t K, int64_t M, int64_t N, void* scratch,
                           int64_t* bad_k, bool* sorted, int64_t* cam_ptr_host, cudaStream_t st) {
  char* sp = static_cast<char*>(scratch);
  unsigned long long* bad = static_cast<unsigned long long*>(carve(sp, sizeof(unsigned long long)));
  int* uns = static_cast<int*>(carve(sp, sizeof(int)));
  int64_t* cptr = static_cast<int64_t*>(carve(sp, sizeof(int64_t) * (size_t)(M + 1)));
  const unsigned long long kk = (unsigned long long)K;
  cudaMemcpyAsync(bad, &kk, sizeof kk, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(uns, 0, sizeof(int), st);
  if (K > 0) k_validate_sorted<<<grid(K), 256, 0, st>>>(d_cam, d_pt, K, M, N, bad, uns, cptr);
  unsigned long long hb = 0;
  int hu = 0;
  cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&hu, uns, sizeof hu, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(cam_ptr_host, cptr, sizeof(int64_t) * (size_t)(M + 1), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) return -1;
  *bad_k = (int64_t)hb;
  *sorted = hu == 0;
  return 0;
}

}  // namespace daba
