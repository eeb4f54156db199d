// coarse.cu — NEXT-3 building block: the Gauss-Newton blocks of the intra-device penalties of the
// coarse-partition surrogate, eq. Ealpha with E' kept exact.  Readings R-N3a (robust weight
// w = rho'(|e|^2), H += w J^T J, g += w J^T r) and R-N3b (world-frame residual r = R e = Pi_v R p, v = l - t,
// Pi_v = I - v v^T / |v|^2) of DESIGN.md §2.  These are the blocks a Schur-complement LM step eliminates:
//   U_i = sum_{k in cam i} w J_c^T J_c (9x9),  g_c,i = sum w J_c^T r,
//   V_j = sum_{k in pt j}  w J_l^T J_l (3x3),  g_l,j = sum w J_l^T r,
//   W_k = w J_c^T J_l (9x3, one per observation),  F = sum_k rho(|r|^2) / 2.
// Product code only: shares nothing with oracle/.  Citations "P:L<n>" are PAPER.md lines.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_math.cuh"

namespace daba {
namespace {

constexpr int kCoarseThreads = 128;
constexpr int kUCols = 45 + 9;  // packed lower triangle of U_i and g_c,i

__device__ __forceinline__ int tri9(int r, int c) { return r * (r + 1) / 2 + c; }  // r >= c

// r, J_c (3x9, row-major), J_l (3x3) of one observation; false if Assumption 2 fails (|l - t| <= eps).
__device__ bool pair_jacobians(const double* __restrict__ cam, const double* __restrict__ l, double2 u, double eps2,
                               double r[3], double Jc[27], double Jl[9]) {
  const double* R = cam;
  const double s = u.x * u.x + u.y * u.y;
  const double b[3] = {1.0, s, s * s};
  const double pz = cam[12] + cam[13] * s + cam[14] * s * s;  // eq. ray
  const double p[3] = {u.x, u.y, pz};
  double q[3], v[3];
  for (int a = 0; a < 3; ++a) {
    q[a] = R[3 * a] * p[0] + R[3 * a + 1] * p[1] + R[3 * a + 2] * p[2];  // R p
    v[a] = l[a] - cam[9 + a];
  }
  const double nv = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  if (!(nv > eps2)) return false;
  const double inv = 1.0 / nv;
  const double lam = (v[0] * q[0] + v[1] * q[1] + v[2] * q[2]) * inv;  // eq. lambdaij
  for (int a = 0; a < 3; ++a) r[a] = q[a] - lam * v[a];              // R e (eq. error)
  // dr/dv = -(v q^T) / |v|^2 - lam I + 2 lam v v^T / |v|^2 = J_l ;  dr/dq = Pi_v
  double Pi[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      const double vv = v[a] * v[c] * inv;
      Pi[3 * a + c] = (a == c ? 1.0 : 0.0) - vv;
      Jl[3 * a + c] = -v[a] * q[c] * inv + 2.0 * lam * vv - (a == c ? lam : 0.0);
    }
  // dq/dtheta = -[q]_x (left perturbation R = Exp(dtheta) R_hat), dq/dd = R e_3 b^T, dv/dt = -I
  const double mq[9] = {0, q[2], -q[1], -q[2], 0, q[0], q[1], -q[0], 0};  // -[q]_x
  for (int a = 0; a < 3; ++a) {
    double Pr3 = 0;
    for (int c = 0; c < 3; ++c) Pr3 += Pi[3 * a + c] * R[3 * c + 2];
    for (int c = 0; c < 3; ++c) {
      Jc[9 * a + c] = Pi[3 * a] * mq[c] + Pi[3 * a + 1] * mq[3 + c] + Pi[3 * a + 2] * mq[6 + c];
      Jc[9 * a + 3 + c] = -Jl[3 * a + c];
      Jc[9 * a + 6 + c] = Pr3 * b[c];
    }
  }
  return true;
}

// One CTA per camera (observations sorted by camera): each thread sums its observations' w J_c^T J_c and
// w J_c^T r in registers, the CTA reduces them in a fixed order; the point blocks go out by fp64 atomics.
template <int LOSS>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_blocks(
    const double* __restrict__ cams, const double* __restrict__ pts, const int32_t* __restrict__ obs_pt,
    const double2* __restrict__ uv, const int64_t* __restrict__ cam_off, double delta, double eps2, double* U,
    double* gc, double* V, double* gl, double* W, double* Fpart) {
  const int i = blockIdx.x;
  __shared__ double scam[15];
  if (threadIdx.x < 15) scam[threadIdx.x] = cams[(size_t)i * 15 + threadIdx.x];
  __syncthreads();
  const double delta2 = delta * delta, idelta2 = 1.0 / delta2;
  double acc[kUCols];
#pragma unroll
  for (int k = 0; k < kUCols; ++k) acc[k] = 0.0;
  double Fsum = 0.0;
  for (int64_t k = cam_off[i] + threadIdx.x; k < cam_off[i + 1]; k += kCoarseThreads) {
    const int32_t j = obs_pt[k];
    const double l[3] = {pts[3 * (size_t)j], pts[3 * (size_t)j + 1], pts[3 * (size_t)j + 2]};
    double r[3], Jc[27], Jl[9];
    double* Wk = W + (size_t)k * 27;
    if (!pair_jacobians(scam, l, uv[k], eps2, r, Jc, Jl)) {  // R-N3d: the pair contributes nothing
      for (int e = 0; e < 27; ++e) Wk[e] = 0.0;
      continue;
    }
    const double sh = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
    double rho = 0.0;
    const double w = loss_eval<LOSS, true>(sh, delta, delta2, idelta2, &rho);  // R-N3a
    Fsum += 0.5 * rho;                                                        // eq. Fij
#pragma unroll
    for (int a = 0; a < 9; ++a) {
#pragma unroll
      for (int c = 0; c <= a; ++c)
        acc[tri9(a, c)] += w * (Jc[a] * Jc[c] + Jc[9 + a] * Jc[9 + c] + Jc[18 + a] * Jc[18 + c]);
      acc[45 + a] += w * (Jc[a] * r[0] + Jc[9 + a] * r[1] + Jc[18 + a] * r[2]);
#pragma unroll
      for (int c = 0; c < 3; ++c)
        Wk[3 * a + c] = w * (Jc[a] * Jl[c] + Jc[9 + a] * Jl[3 + c] + Jc[18 + a] * Jl[6 + c]);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int c = 0; c <= a; ++c)
        atomicAdd(V + 9 * (size_t)j + 3 * a + c, w * (Jl[a] * Jl[c] + Jl[3 + a] * Jl[3 + c] + Jl[6 + a] * Jl[6 + c]));
      atomicAdd(gl + 3 * (size_t)j + a, w * (Jl[a] * r[0] + Jl[3 + a] * r[1] + Jl[6 + a] * r[2]));
    }
  }
  // CTA reduction, fixed order: warp shuffles, then the four warps' rows in order
  __shared__ double red[kCoarseThreads / 32][kUCols + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kUCols; ++k) {
    double x = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
    if (lane == 0) red[warp][k] = x;
  }
  {
    double x = Fsum;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
    if (lane == 0) red[warp][kUCols] = x;
  }
  __syncthreads();
  for (int k = threadIdx.x; k <= kUCols; k += kCoarseThreads) {
    double x = 0.0;
    for (int w = 0; w < kCoarseThreads / 32; ++w) x += red[w][k];
    if (k < 45) {
      int a = 0;
      while (tri9(a + 1, 0) <= k) ++a;
      const int c = k - tri9(a, 0);
      U[(size_t)i * 81 + 9 * a + c] = x;
      U[(size_t)i * 81 + 9 * c + a] = x;
    } else if (k < kUCols) {
      gc[(size_t)i * 9 + (k - 45)] = x;
    } else {
      Fpart[i] = x;
    }
  }
}

// V_j symmetric: the atomics filled the lower triangle; mirror it.
__global__ void k_coarse_mirror(double* V, int64_t N) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  double* v = V + 9 * j;
  v[1] = v[3];
  v[2] = v[6];
  v[5] = v[7];
}

}  // namespace
}  // namespace daba

extern "C" int daba_coarse_blocks(const double* cams, int64_t M, const double* pts, int64_t N,
                                  const int32_t* obs_pt, const double* obs_uv, const int64_t* cam_off, int64_t K,
                                  int loss, double scale, double eps, double* U, double* gc, double* V, double* gl,
                                  double* W, double* F_cam, void* stream) {
  using namespace daba;
  if (M < 0 || N < 0 || K < 0 || M > INT32_MAX || !(scale > 0) || !(eps >= 0) || loss < 0 || loss > 2) return -1;
  if ((M > 0 && (!cams || !cam_off || !U || !gc || !F_cam)) || (N > 0 && (!pts || !V || !gl)) ||
      (K > 0 && (!obs_pt || !obs_uv || !W)))
    return -1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (N > 0) {
    if (cudaMemsetAsync(V, 0, (size_t)N * 9 * sizeof(double), st) != cudaSuccess) return -3;
    if (cudaMemsetAsync(gl, 0, (size_t)N * 3 * sizeof(double), st) != cudaSuccess) return -3;
  }
  if (M > 0) {
    const double2* uv = reinterpret_cast<const double2*>(obs_uv);
    const double eps2 = eps * eps;
    const dim3 g((unsigned)M), b(kCoarseThreads);
    if (loss == kHuber)
      k_coarse_blocks<kHuber><<<g, b, 0, st>>>(cams, pts, obs_pt, uv, cam_off, scale, eps2, U, gc, V, gl, W, F_cam);
    else if (loss == kCauchy)
      k_coarse_blocks<kCauchy><<<g, b, 0, st>>>(cams, pts, obs_pt, uv, cam_off, scale, eps2, U, gc, V, gl, W, F_cam);
    else
      k_coarse_blocks<kTrivial><<<g, b, 0, st>>>(cams, pts, obs_pt, uv, cam_off, scale, eps2, U, gc, V, gl, W, F_cam);
  }
  if (N > 0) k_coarse_mirror<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(V, N);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
