// device_math.cuh — fp64 device helpers of the DABA hot path (sm_100a).
//
// Product code only: shares nothing with oracle/.  Citations "P:L<n>" are PAPER.md lines.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace daba {

enum LossKind { kTrivial = 0, kHuber = 1, kCauchy = 2 };

// 1/x and 1/sqrt(x) for the per-observation hot loops: the MUFU seed refined by two Newton steps (quadratic: the
// ~23-bit seed reaches the fp64 rounding level), within 1 ulp of the correctly rounded result for positive normal
// x, without the range check and slow path of __drcp_rn / rsqrt (camera pass 0.717 -> 0.709 ms on Final-13682).
__device__ __forceinline__ double rcp_d(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_d(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;  // y <- y (3 - x y^2) / 2, twice
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}

// log(1 + q) for q >= 0 (the Cauchy loss's rho at every observation of the x^k anchor): q < sqrt(2) - 1 takes
// f = q / (2 + q) directly (no rounding of 1 + q), larger q reduces 1 + q = m 2^e with m in [sqrt(1/2), sqrt(2))
// and f = (m - 1) / (m + 1); then log1p = e ln 2 + 2 atanh(f), the atanh series to f^21 (|f| <= 0.1716, so the
// first omitted term is below 2^-53 of the sum).  Within a few ulp of the correctly rounded value; about a third of
// the FP64 instructions of the library log1p (camera pass on the Cauchy slab: see DESIGN.md §6).  NaN / inf (and
// negative q, which the loss never passes) go to the library routine.
__device__ __forceinline__ double log1p_pos(double q) {
  if (!(q >= 0.0 && q <= 1.7976931348623157e308)) return log1p(q);
  const double u = 1.0 + q;
  const int hi = __double2hiint(u);
  int e = (hi >> 20) - 1023;
  double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(u));  // [1, 2)
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const bool small = q < 0.41421356237309503;
  const double num = small ? q : m - 1.0;
  const double den = small ? 2.0 + q : m + 1.0;
  const double f = num * rcp_d(den);
  const double z = f * f;
  double P = 1.0 / 21;
  P = fma(P, z, 1.0 / 19);
  P = fma(P, z, 1.0 / 17);
  P = fma(P, z, 1.0 / 15);
  P = fma(P, z, 1.0 / 13);
  P = fma(P, z, 1.0 / 11);
  P = fma(P, z, 1.0 / 9);
  P = fma(P, z, 1.0 / 7);
  P = fma(P, z, 1.0 / 5);
  P = fma(P, z, 1.0 / 3);
  const double f2 = f + f;
  const double lm = fma(f2 * z, P, f2);  // 2 atanh(f) = log m
  const double de = small ? 0.0 : (double)e;
  return fma(de, 6.93147180369123816490e-01, fma(de, 1.90821492927058770002e-10, lm));  // ln 2 = hi + lo
}

// Robust loss of eq. Fij, Assumption 1; delta2 = delta^2, idelta2 = 1/delta^2.
// Returns w = rho'(s) and, when WANT_RHO, rho(s).
template <int LOSS, bool WANT_RHO>
__device__ __forceinline__ double loss_eval(double s, double delta, double delta2, double idelta2, double* rho) {
  if (LOSS == kHuber) {
    if (s <= delta2) {
      if (WANT_RHO) *rho = s;
      return 1.0;
    }
    const double ri = rsqrt_d(s);
    if (WANT_RHO) *rho = 2.0 * delta * (s * ri) - delta2;
    return delta * ri;
  } else if (LOSS == kCauchy) {
    const double q = s * idelta2;
#ifndef DABA_LIB_LOG1P
    if (WANT_RHO) *rho = delta2 * log1p_pos(q);
#else
    if (WANT_RHO) *rho = delta2 * log1p(q);
#endif
    return rcp_d(1.0 + q);  // = 1 / (1 + q) without the division's slow-path call
  } else {
    if (WANT_RHO) *rho = s;
    return 1.0;
  }
}

struct M3 {
  double a[9];
};

__device__ __forceinline__ void mat3_mul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) C[3 * r + c] = fma(A[3 * r], B[c], fma(A[3 * r + 1], B[3 + c], A[3 * r + 2] * B[6 + c]));
}
// C = A^T B
__device__ __forceinline__ void mat3_tmul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) C[3 * r + c] = fma(A[r], B[c], fma(A[3 + r], B[3 + c], A[6 + r] * B[6 + c]));
}
__device__ __forceinline__ double det3(const double* A) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) + A[2] * (A[3] * A[7] - A[4] * A[6]);
}

// Exp(w) - I for w in so(3) (Rodrigues, accurate for small |w|), row-major.
__device__ __forceinline__ void expm_minus_identity(const double* w, double* E) {
  const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  double a, b;
  if (th2 < 1e-4) {
    // |th| < 1e-2 (LM steps): Taylor series of sin(th)/th and (1 - cos th)/th^2, truncation < 1e-20 relative
    a = 1.0 + th2 * (-1.0 / 6.0 + th2 * (1.0 / 120.0 + th2 * (-1.0 / 5040.0 + th2 * (1.0 / 362880.0))));
    b = 0.5 + th2 * (-1.0 / 24.0 + th2 * (1.0 / 720.0 + th2 * (-1.0 / 40320.0 + th2 * (1.0 / 3628800.0))));
  } else {
    const double th = sqrt(th2);
    a = sin(th) / th;
    // 1 - cos(th) = 2 sin^2(th/2), no cancellation
    const double sh = sin(0.5 * th);
    b = 2.0 * sh * sh / th2;
  }
  const double x = w[0], y = w[1], z = w[2];
  // a [w]x + b [w]x^2,  [w]x^2 = w w^T - th2 I
  E[0] = b * (x * x - th2);
  E[1] = -a * z + b * x * y;
  E[2] = a * y + b * x * z;
  E[3] = a * z + b * x * y;
  E[4] = b * (y * y - th2);
  E[5] = -a * x + b * y * z;
  E[6] = -a * y + b * x * z;
  E[7] = a * x + b * y * z;
  E[8] = b * (z * z - th2);
}

// Symmetric 3x3 eigen-decomposition by cyclic Jacobi rotations: S = V diag(lam) V^T (columns of V).
__device__ inline void sym3_eig(const double* Sin, double* lam, double* V) {
  double S[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) S[k] = Sin[k];
#pragma unroll
  for (int k = 0; k < 9; ++k) V[k] = (k % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = fabs(S[1]) + fabs(S[2]) + fabs(S[5]);
    const double diag = fabs(S[0]) + fabs(S[4]) + fabs(S[8]);
    if (off <= 1e-18 * diag || off == 0.0) break;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double apq = S[3 * p + q];
      if (apq == 0.0) continue;
      const double theta = (S[3 * q + q] - S[3 * p + p]) / (2.0 * apq);
      const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
      // S <- J^T S J with J the (p,q) rotation
      for (int k = 0; k < 3; ++k) {
        const double skp = S[3 * k + p], skq = S[3 * k + q];
        S[3 * k + p] = c * skp - s * skq;
        S[3 * k + q] = s * skp + c * skq;
      }
      for (int k = 0; k < 3; ++k) {
        const double spk = S[3 * p + k], sqk = S[3 * q + k];
        S[3 * p + k] = c * spk - s * sqk;
        S[3 * q + k] = s * spk + c * sqk;
      }
      for (int k = 0; k < 3; ++k) {
        const double vkp = V[3 * k + p], vkq = V[3 * k + q];
        V[3 * k + p] = c * vkp - s * vkq;
        V[3 * k + q] = s * vkp + c * vkq;
      }
    }
  }
  lam[0] = S[0];
  lam[1] = S[4];
  lam[2] = S[8];
}

// ProjRot3D(M) = argmin_{R in SO(3)} ||R - M||_F^2 (eq. proj_rot3d).
// det(M) > 0: the orthogonal polar factor of M, by Newton's iteration X <- (X + X^{-T}) / 2 (quadratic
// convergence from the near-rotations extrapolation produces).  Otherwise: from M^T M = V diag(sig^2) V^T,
// R = u1 v1^T + u2 v2^T + det(V) (u1 x u2) v3^T with u_k = M v_k / sig_k, sig1 >= sig2 >= sig3 — the SVD formula
// U diag(1,1,det(U V^T)) V^T with the sign flip on the smallest singular direction.
__device__ inline void proj_rot3d(const double* M, double* R) {
  const double dM = det3(M);
  if (dM > 0) {
    double X[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) X[k] = M[k];
    for (int it = 0; it < 40; ++it) {
      const double d = det3(X);
      const double id = 1.0 / d;
      // X^{-T} = cofactor(X) / det
      double C[9];
      C[0] = (X[4] * X[8] - X[5] * X[7]) * id;
      C[1] = (X[5] * X[6] - X[3] * X[8]) * id;
      C[2] = (X[3] * X[7] - X[4] * X[6]) * id;
      C[3] = (X[2] * X[7] - X[1] * X[8]) * id;
      C[4] = (X[0] * X[8] - X[2] * X[6]) * id;
      C[5] = (X[1] * X[6] - X[0] * X[7]) * id;
      C[6] = (X[1] * X[5] - X[2] * X[4]) * id;
      C[7] = (X[2] * X[3] - X[0] * X[5]) * id;
      C[8] = (X[0] * X[4] - X[1] * X[3]) * id;
      double diff = 0;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const double nx = 0.5 * (X[k] + C[k]);
        diff = fmax(diff, fabs(nx - X[k]));
        X[k] = nx;
      }
      if (diff <= 1e-15) break;
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = X[k];
    return;
  }
  double MtM[9], lam[3], V[9];
  mat3_tmul(M, M, MtM);
  sym3_eig(MtM, lam, V);
  int o[3] = {0, 1, 2};
  if (lam[o[1]] > lam[o[0]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
  if (lam[o[2]] > lam[o[1]]) { int t = o[1]; o[1] = o[2]; o[2] = t; }
  if (lam[o[1]] > lam[o[0]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
  double v[3][3], u[2][3];
  for (int k = 0; k < 3; ++k)
    for (int r = 0; r < 3; ++r) v[k][r] = V[3 * r + o[k]];
  for (int k = 0; k < 2; ++k) {
    double x[3];
    for (int r = 0; r < 3; ++r) x[r] = M[3 * r] * v[k][0] + M[3 * r + 1] * v[k][1] + M[3 * r + 2] * v[k][2];
    const double n = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
    for (int r = 0; r < 3; ++r) u[k][r] = n > 0 ? x[r] / n : (r == k ? 1.0 : 0.0);
  }
  const double u3[3] = {u[0][1] * u[1][2] - u[0][2] * u[1][1], u[0][2] * u[1][0] - u[0][0] * u[1][2],
                        u[0][0] * u[1][1] - u[0][1] * u[1][0]};
  const double Vm[9] = {v[0][0], v[1][0], v[2][0], v[0][1], v[1][1], v[2][1], v[0][2], v[1][2], v[2][2]};
  const double sV = det3(Vm) < 0 ? -1.0 : 1.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R[3 * r + c] = u[0][r] * v[0][c] + u[1][r] * v[1][c] + sV * u3[r] * v[2][c];
}

}  // namespace daba
