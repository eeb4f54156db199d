// oracle/daba_oracle.cpp — plain, slow, single-threaded CPU oracle of one DABA iteration.
//
// TEST INFRASTRUCTURE ONLY (see daba_oracle.h).  No BLAS, no OpenMP, no SIMD tricks,
// no code shared with the CUDA product path.  Every function cites the PAPER.md
// passage it follows ("P:L<n>" = /root/reference/PAPER.md line n).  Readings of
// passages the paper leaves open are SURVEY.md §8(c) Q1-Q23, restated in DESIGN.md.
//
// Summation order: per-camera and per-point sums run over that camera's / point's
// observations in ascending input order; global sums are Kahan-compensated sums
// over per-camera / per-point partials.
#include "daba_oracle.h"

#include <cmath>
#include <cstring>
#include <new>
#include <vector>

namespace {

// ---------------------------------------------------------------- small linear algebra
void mat_vec(const double* A, const double* x, double* y) {  // y = A x (3x3)
  for (int r = 0; r < 3; ++r) y[r] = A[3 * r] * x[0] + A[3 * r + 1] * x[1] + A[3 * r + 2] * x[2];
}
void mat_t_vec(const double* A, const double* x, double* y) {  // y = A^T x
  for (int c = 0; c < 3; ++c) y[c] = A[c] * x[0] + A[3 + c] * x[1] + A[6 + c] * x[2];
}
void mat_mul(const double* A, const double* B, double* C) {  // C = A B
  double T[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += A[3 * r + k] * B[3 * k + c];
      T[3 * r + c] = s;
    }
  std::memcpy(C, T, sizeof T);
}
double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
double det3(const double* A) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) + A[2] * (A[3] * A[7] - A[4] * A[6]);
}

struct Kahan {  // compensated summation for global sums
  double s = 0, c = 0;
  void add(double x) {
    const double y = x - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
  }
};

// Per-observation coefficients of Proposition 1 at an anchor.
struct Coef {
  bool degenerate;  // Assumption 2 violated at this anchor: pair contributes nothing (Q17)
  double p[3];      // undistorted ray at the anchor intrinsics, eq. ray
  double b[3];      // (1, |u|^2, |u|^4): d p_z / d d
  double lambda;    // eq. gamma
  double Re[3];     // R e: the reprojection error, eq. error, rotated to the world frame
  double s_hat;     // ||e||^2
  double rho, w, a; // rho(||e||^2), eq. w, eq. a
};

Coef coefficients(const double* cam, const double* l, const double* u, const orc_options* o) {
  Coef c{};
  const double* R = cam;
  const double* t = cam + 9;
  const double* d = cam + 12;
  orc_ray(d, u, c.p);
  const double s = u[0] * u[0] + u[1] * u[1];
  c.b[0] = 1.0;
  c.b[1] = s;
  c.b[2] = s * s;
  double e[3];
  if (orc_optimal_scale(R, t, l, c.p, o->eps, &c.lambda) != 0 ||
      orc_reprojection_error(R, t, l, c.p, o->eps, e) != 0) {
    c.degenerate = true;
    c.lambda = 0;
    return c;
  }
  mat_vec(R, e, c.Re);
  c.s_hat = dot3(e, e);
  orc_loss(o->kind, o->scale, c.s_hat, &c.rho, &c.w);
  c.a = 0.5 * c.rho - 0.5 * c.w * c.s_hat;  // eq. a
  return c;
}

// ---------------------------------------------------------------- 9x9 LM step (D3 / Q3)
// Jacobian of r(c) = R p(d) + lambda t - g (the vector inside P_ij, eq. P) w.r.t. the
// tangent (dtheta, dt, dd) at the anchor, left perturbation R = Exp(dtheta) R_hat (Q5):
//   dr/dtheta = -[R_hat p_hat]_x,  dr/dt = lambda I,  dr/dd = R_hat e_3 b^T.
void camera_jacobian(const double* cam, const Coef& c, double J[27]) {
  const double* R = cam;
  double Rp[3];
  mat_vec(R, c.p, Rp);
  // -[a]_x = [[0, a3, -a2], [-a3, 0, a1], [a2, -a1, 0]]
  const double S[9] = {0, Rp[2], -Rp[1], -Rp[2], 0, Rp[0], Rp[1], -Rp[0], 0};
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) J[9 * r + k] = S[3 * r + k];
    for (int k = 0; k < 3; ++k) J[9 * r + 3 + k] = (r == k) ? c.lambda : 0.0;
    for (int k = 0; k < 3; ++k) J[9 * r + 6 + k] = R[3 * r + 2] * c.b[k];
  }
}

void build_normal_equations(const double* cam, const std::vector<Coef>& co, const orc_options* o, double H[81],
                            double g[9]) {
  for (int i = 0; i < 81; ++i) H[i] = 0;
  for (int i = 0; i < 9; ++i) g[i] = 0;
  double J[27];
  for (const Coef& c : co) {
    if (c.degenerate) continue;
    camera_jacobian(cam, c, J);
    // P = w ||r||^2 + a/2 with r_hat = (R_hat e)/2 at the anchor:
    //   Gauss-Newton Hessian 2 w J^T J, gradient 2 w J^T r_hat = w J^T (R_hat e).
    for (int i = 0; i < 9; ++i) {
      for (int j = 0; j < 9; ++j) {
        double s = 0;
        for (int r = 0; r < 3; ++r) s += J[9 * r + i] * J[9 * r + j];
        H[9 * i + j] += 2.0 * c.w * s;
      }
      double s = 0;
      for (int r = 0; r < 3; ++r) s += J[9 * r + i] * c.Re[r];
      g[i] += c.w * s;
    }
  }
  // proximal term xi/2 (||R - R_hat||_F^2 + ||t - t_hat||^2 + ||d - d_hat||^2) (eq. Ealpha, Q7):
  // ||Exp(dtheta) - I||_F^2 = 2 ||dtheta||^2 + O(|dtheta|^3), zero gradient at the anchor (Q13).
  for (int i = 0; i < 9; ++i) H[9 * i + i] += o->xi * (i < 3 ? 2.0 : 1.0);
}

// Decrease of sum_j P_j + xi/2 ||c - c_hat||^2 from the anchor to trial c'.  Anchor-relative form
// (Q21): P_j(c') - P_j(c_hat) = w dr.(dr + R_hat e), dr = R' p(d') - R_hat p_hat + lambda (t' - t_hat),
// which is eq. P expanded around r_hat = R_hat e / 2.
double camera_decrease(const double* anchor, const double* trial, const std::vector<Coef>& co, const double* u_list,
                       const orc_options* o) {
  const double* Rh = anchor;
  const double* th = anchor + 9;
  const double* R2 = trial;
  const double* t2 = trial + 9;
  const double* d2 = trial + 12;
  double sum = 0;
  for (size_t j = 0; j < co.size(); ++j) {
    const Coef& c = co[j];
    if (c.degenerate) continue;
    double p2[3], Rp2[3], Rph[3];
    orc_ray(d2, u_list + 2 * j, p2);
    mat_vec(R2, p2, Rp2);
    mat_vec(Rh, c.p, Rph);
    double dr[3];
    for (int r = 0; r < 3; ++r) dr[r] = (Rp2[r] - Rph[r]) + c.lambda * (t2[r] - th[r]);
    double q = 0;
    for (int r = 0; r < 3; ++r) q += dr[r] * (dr[r] + c.Re[r]);
    sum += c.w * q;
  }
  double prox = 0;
  for (int i = 0; i < 15; ++i) prox += (trial[i] - anchor[i]) * (trial[i] - anchor[i]);
  return sum + 0.5 * o->xi * prox;
}

// Cholesky of a 9x9 SPD matrix; false on a non-positive pivot (Q3: a failed trial).
bool cholesky9(const double* A, double* L) {
  for (int i = 0; i < 81; ++i) L[i] = 0;
  for (int j = 0; j < 9; ++j) {
    double s = A[9 * j + j];
    for (int k = 0; k < j; ++k) s -= L[9 * j + k] * L[9 * j + k];
    if (!(s > 0)) return false;
    L[9 * j + j] = std::sqrt(s);
    for (int i = j + 1; i < 9; ++i) {
      double t = A[9 * i + j];
      for (int k = 0; k < j; ++k) t -= L[9 * i + k] * L[9 * j + k];
      L[9 * i + j] = t / L[9 * j + j];
    }
  }
  return true;
}
void cholesky_solve9(const double* L, const double* b, double* x) {
  double y[9];
  for (int i = 0; i < 9; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[9 * i + k] * y[k];
    y[i] = s / L[9 * i + i];
  }
  for (int i = 8; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 9; ++k) s -= L[9 * k + i] * x[k];
    x[i] = s / L[9 * i + i];
  }
}

// One successful LM step on the camera subproblem ("only one successful inner LM step"; Q3):
// Marquardt damping H + mu diag(H), mu = mu0 * mu_up^tau, tau = 0..T-1, solved by Jacobi-scaled Cholesky
// (D3); accept the first trial with a strict decrease, otherwise keep the anchor.
void camera_lm(const double* anchor, const std::vector<Coef>& co, const double* u_list, const orc_options* o,
               double* out, int* trial, double* dP) {
  double H[81], g[9];
  build_normal_equations(anchor, co, o, H, g);
  double sc[9];
  for (int i = 0; i < 9; ++i) sc[i] = 1.0 / std::sqrt(H[9 * i + i]);
  double Hs[81], gs[9];
  for (int i = 0; i < 9; ++i) {
    gs[i] = g[i] * sc[i];
    for (int j = 0; j < 9; ++j) Hs[9 * i + j] = H[9 * i + j] * sc[i] * sc[j];
  }
  std::memcpy(out, anchor, 15 * sizeof(double));
  *trial = -1;
  *dP = 0;
  double mu = o->lm_mu0;
  for (int tau = 0; tau < o->lm_max_trials; ++tau, mu *= o->lm_mu_up) {
    double A[81], L[81];
    std::memcpy(A, Hs, sizeof A);
    for (int i = 0; i < 9; ++i) A[9 * i + i] += mu * Hs[9 * i + i];  // (H + mu diag H), scaled
    if (!cholesky9(A, L)) continue;
    double ng[9], y[9];
    for (int i = 0; i < 9; ++i) ng[i] = -gs[i];
    cholesky_solve9(L, ng, y);
    double delta[9];
    for (int i = 0; i < 9; ++i) delta[i] = y[i] * sc[i];
    double c2[15], E[9];
    orc_expmap(delta, E);
    mat_mul(E, anchor, c2);  // R' = Exp(dtheta) R_hat (Q5)
    for (int k = 0; k < 3; ++k) c2[9 + k] = anchor[9 + k] + delta[3 + k];
    for (int k = 0; k < 3; ++k) c2[12 + k] = anchor[12 + k] + delta[6 + k];
    const double dec = camera_decrease(anchor, c2, co, u_list, o);
    if (dec < 0) {
      std::memcpy(out, c2, sizeof c2);
      *trial = tau;
      *dP = dec;
      return;
    }
  }
}

// Exact minimiser of sum_i Q_ij(l) + xi/2 ||l - l_hat||^2 (eq. Q P:L210-212 with eq. Ealpha):
// Q_ij(l_hat + dl) = w ||lambda dl - R_hat e / 2||^2 + a/2, so the stationarity condition is
// (2 sum w lambda^2 + xi) dl = sum w lambda R_hat e  (Q4: exact, Assumption 4 holds for points).
void point_closed_form(const double* l_hat, const std::vector<Coef>& co, const orc_options* o, double* out) {
  double A = 0, C[3] = {0, 0, 0};
  for (const Coef& c : co) {
    if (c.degenerate) continue;
    A += c.w * c.lambda * c.lambda;
    for (int r = 0; r < 3; ++r) C[r] += c.w * c.lambda * c.Re[r];
  }
  const double den = 2.0 * A + o->xi;
  for (int r = 0; r < 3; ++r) out[r] = l_hat[r] + C[r] / den;
}

// Decrease of sum_i Q_ij + xi/2 ||l - l_hat||^2 from the anchor to l (anchor-relative form of eq. Q).
double point_decrease(const double* l_hat, const double* l, const std::vector<Coef>& co, const orc_options* o) {
  double dl[3] = {l[0] - l_hat[0], l[1] - l_hat[1], l[2] - l_hat[2]};
  double sum = 0;
  for (const Coef& c : co) {
    if (c.degenerate) continue;
    double q = 0;
    for (int r = 0; r < 3; ++r) q += c.lambda * dl[r] * (c.lambda * dl[r] - c.Re[r]);
    sum += c.w * q;
  }
  return sum + 0.5 * o->xi * dot3(dl, dl);
}

// Per-pair anchor-relative changes of P_ij and Q_ij (eq. P, eq. Q expanded around the anchor, Q21), without
// the proximal term: P_ij(c|x_hat) - P_ij(c_hat|x_hat) = w dr.(dr + R_hat e),
// Q_ij(l|x_hat) - Q_ij(l_hat|x_hat) = w (lambda dl).(lambda dl - R_hat e).
double pair_dP(const double* anchor, const double* cam, const Coef& c, const double* u) {
  if (c.degenerate) return 0.0;
  double p2[3], Rp2[3], Rph[3], dr[3];
  orc_ray(cam + 12, u, p2);
  mat_vec(cam, p2, Rp2);
  mat_vec(anchor, c.p, Rph);
  for (int r = 0; r < 3; ++r) dr[r] = (Rp2[r] - Rph[r]) + c.lambda * (cam[9 + r] - anchor[9 + r]);
  double q = 0;
  for (int r = 0; r < 3; ++r) q += dr[r] * (dr[r] + c.Re[r]);
  return c.w * q;
}
double pair_dQ(const double* l_hat, const double* l, const Coef& c) {
  if (c.degenerate) return 0.0;
  double q = 0;
  for (int r = 0; r < 3; ++r) {
    const double x = c.lambda * (l[r] - l_hat[r]);
    q += x * (x - c.Re[r]);
  }
  return c.w * q;
}

}  // namespace

// ================================================================ geometry (§3)
extern "C" void orc_ray(const double d[3], const double u[2], double p[3]) {
  // eq. ray: p = (u, d1 + d2 |u|^2 + d3 |u|^4)
  const double s = u[0] * u[0] + u[1] * u[1];
  p[0] = u[0];
  p[1] = u[1];
  p[2] = d[0] + d[1] * s + d[2] * s * s;
}

extern "C" int orc_optimal_scale(const double R[9], const double t[3], const double l[3], const double p[3],
                                 double eps, double* lambda) {
  // eq. lambdaij: lambda = (l - t)^T R p / ||l - t||^2, unique when ||l - t|| != 0 (Assumption 2)
  const double v[3] = {l[0] - t[0], l[1] - t[1], l[2] - t[2]};
  const double nv = dot3(v, v);
  if (!(nv > eps * eps)) return -1;
  double Rp[3];
  mat_vec(R, p, Rp);
  *lambda = dot3(v, Rp) / nv;
  return 0;
}

extern "C" int orc_reprojection_error(const double R[9], const double t[3], const double l[3], const double p[3],
                                      double eps, double e[3]) {
  // eq. error: e = (I - R^T (l-t)(l-t)^T R / ||l-t||^2) p
  const double v[3] = {l[0] - t[0], l[1] - t[1], l[2] - t[2]};
  const double nv = dot3(v, v);
  if (!(nv > eps * eps)) return -1;
  double Rtv[3];
  mat_t_vec(R, v, Rtv);  // R^T (l - t)
  const double proj = dot3(Rtv, p) / nv;
  for (int r = 0; r < 3; ++r) e[r] = p[r] - Rtv[r] * proj;
  return 0;
}

extern "C" void orc_loss(int kind, double scale, double s, double* rho, double* drho) {
  // Robust losses satisfying Assumption 1; thresholds are reading Q9 (delta in ||e|| units).
  const double d2 = scale * scale;
  if (kind == ORC_LOSS_HUBER) {
    if (s <= d2) {
      *rho = s;
      *drho = 1.0;
    } else {
      const double r = std::sqrt(s);
      *rho = 2.0 * scale * r - d2;
      *drho = scale / r;
    }
  } else if (kind == ORC_LOSS_CAUCHY) {
    *rho = d2 * std::log1p(s / d2);
    *drho = 1.0 / (1.0 + s / d2);
  } else {
    *rho = s;
    *drho = 1.0;
  }
}

extern "C" int orc_penalty(const double cam[15], const double l[3], const double u[2], int kind, double scale,
                           double eps, double* F) {
  // eq. Fij: F_ij = rho(||e_ij||^2) / 2
  double p[3], e[3];
  orc_ray(cam + 12, u, p);
  if (orc_reprojection_error(cam, cam + 9, l, p, eps, e) != 0) return -1;
  double rho, drho;
  orc_loss(kind, scale, dot3(e, e), &rho, &drho);
  *F = 0.5 * rho;
  return 0;
}

// ================================================================ surrogate (§4)
extern "C" int orc_coefficients(const double cam[15], const double l[3], const double u[2], int kind, double scale,
                                double eps, double* a, double* w, double* lambda, double g[3]) {
  // Proposition 1: a (eq. a), w (eq. w), lambda (eq. gamma), g (eq. g) at the anchor.
  orc_options o{};
  o.kind = kind;
  o.scale = scale;
  o.eps = eps;
  const Coef c = coefficients(cam, l, u, &o);
  if (c.degenerate) return -1;
  *a = c.a;
  *w = c.w;
  *lambda = c.lambda;
  double Rp[3];
  mat_vec(cam, c.p, Rp);
  for (int r = 0; r < 3; ++r) g[r] = 0.5 * Rp[r] + 0.5 * c.lambda * cam[9 + r] + 0.5 * c.lambda * l[r];  // eq. g
  return 0;
}

extern "C" double orc_P(double a, double w, double lambda, const double g[3], const double cam[15],
                        const double u[2]) {
  // eq. P: P_ij(c) = w ||R p + lambda t - g||^2 + a/2
  double p[3], Rp[3];
  orc_ray(cam + 12, u, p);
  mat_vec(cam, p, Rp);
  double s = 0;
  for (int r = 0; r < 3; ++r) {
    const double x = Rp[r] + lambda * cam[9 + r] - g[r];
    s += x * x;
  }
  return w * s + 0.5 * a;
}

extern "C" double orc_Q(double a, double w, double lambda, const double g[3], const double l[3]) {
  // eq. Q: Q_ij(l) = w ||lambda l - g||^2 + a/2
  double s = 0;
  for (int r = 0; r < 3; ++r) {
    const double x = lambda * l[r] - g[r];
    s += x * x;
  }
  return w * s + 0.5 * a;
}

// ================================================================ acceleration (§5)
extern "C" void orc_proj_rot3d(const double Min[9], double Rout[9]) {
  // eq. proj_rot3d: argmin_{R in SO(3)} ||R - M||^2, closed form via the SVD M = U S V^T
  // (Umeyama): R = U diag(1, 1, det(U V^T)) V^T, sign flip on the smallest singular direction (Q14).
  // SVD by one-sided Jacobi rotations on the columns of M.
  double A[9], V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  std::memcpy(A, Min, sizeof A);
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double alpha = 0, beta = 0, gam = 0;
        for (int i = 0; i < 3; ++i) {
          alpha += A[3 * i + p] * A[3 * i + p];
          beta += A[3 * i + q] * A[3 * i + q];
          gam += A[3 * i + p] * A[3 * i + q];
        }
        if (gam == 0.0 || std::fabs(gam) <= 1e-300) continue;
        const double conv = std::fabs(gam) / std::sqrt(alpha * beta);
        if (!(conv > 1e-17)) continue;
        off = std::fmax(off, conv);
        const double zeta = (beta - alpha) / (2.0 * gam);
        const double tt = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + tt * tt), s = c * tt;
        for (int i = 0; i < 3; ++i) {
          const double ap = A[3 * i + p], aq = A[3 * i + q];
          A[3 * i + p] = c * ap - s * aq;
          A[3 * i + q] = s * ap + c * aq;
          const double vp = V[3 * i + p], vq = V[3 * i + q];
          V[3 * i + p] = c * vp - s * vq;
          V[3 * i + q] = s * vp + c * vq;
        }
      }
    if (off < 1e-16) break;
  }
  // singular values = column norms of A; U columns = normalised columns; sort descending
  double sig[3];
  int ord[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) sig[k] = std::sqrt(A[k] * A[k] + A[3 + k] * A[3 + k] + A[6 + k] * A[6 + k]);
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (sig[ord[j]] > sig[ord[i]]) {
        const int tmp = ord[i];
        ord[i] = ord[j];
        ord[j] = tmp;
      }
  double U[9], Vs[9];
  for (int k = 0; k < 3; ++k) {
    const int c = ord[k];
    for (int i = 0; i < 3; ++i) Vs[3 * i + k] = V[3 * i + c];
    for (int i = 0; i < 3; ++i) U[3 * i + k] = sig[c] > 0 ? A[3 * i + c] / sig[c] : 0.0;
  }
  if (!(sig[ord[2]] > 1e-300 * (sig[ord[0]] + 1e-300))) {  // rank-deficient: complete U by a cross product
    U[2] = U[3] * U[7] - U[6] * U[4];
    U[5] = U[6] * U[1] - U[0] * U[7];
    U[8] = U[0] * U[4] - U[3] * U[1];
  }
  double Vt[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Vt[3 * i + j] = Vs[3 * j + i];
  double UVt[9];
  mat_mul(U, Vt, UVt);
  const double dsgn = det3(UVt) < 0 ? -1.0 : 1.0;
  for (int i = 0; i < 3; ++i) U[3 * i + 2] *= dsgn;
  mat_mul(U, Vt, Rout);
}

extern "C" void orc_schedule(double s, double* s_next, double* gamma) {
  // eq. nesterov_scalar, Algorithm 1 line 407 order (Q11):
  // s^{(k+1)} = (sqrt(4 s^{(k)2} + 1) + 1) / 2,  gamma^{(k)} = (s^{(k)} - 1) / s^{(k+1)}
  *s_next = (std::sqrt(4.0 * s * s + 1.0) + 1.0) / 2.0;
  *gamma = (s - 1.0) / *s_next;
}

extern "C" void orc_expmap(const double w[3], double R[9]) {
  // Rodrigues' formula; series below 1e-8 rad (Q5)
  const double th2 = dot3(w, w), th = std::sqrt(th2);
  double a, b;
  if (th < 1e-8) {
    a = 1.0 - th2 / 6.0;
    b = 0.5 - th2 / 24.0;
  } else {
    a = std::sin(th) / th;
    b = (1.0 - std::cos(th)) / th2;
  }
  const double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double K2[9];
  mat_mul(K, K, K2);
  for (int i = 0; i < 9; ++i) R[i] = (i % 4 == 0 ? 1.0 : 0.0) + a * K[i] + b * K2[i];
}

extern "C" void orc_bal_to_native(const double bal[9], double cam[15]) {
  // BAL: x_cam = R_w2c x + t_w2c.  Paper: x_cam = R^T (l - t)  =>  R = R_w2c^T, t = -R t_w2c.
  double Rw2c[9];
  orc_expmap(bal, Rw2c);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) cam[3 * i + j] = Rw2c[3 * j + i];
  double t[3];
  mat_vec(cam, bal + 3, t);
  for (int k = 0; k < 3; ++k) cam[9 + k] = -t[k];
  // d = (f, f k1, f k2)
  cam[12] = bal[6];
  cam[13] = bal[6] * bal[7];
  cam[14] = bal[6] * bal[8];
}

extern "C" void orc_native_to_bal(const double cam[15], double bal[9]) {
  // Inverse of orc_bal_to_native.  Angle-axis of R_w2c = R^T through its quaternion.
  const double* R = cam;
  const double Q[9] = {R[0], R[3], R[6], R[1], R[4], R[7], R[2], R[5], R[8]};  // R_w2c
  const double tr = Q[0] + Q[4] + Q[8];
  double q[4];
  if (tr > Q[0] && tr > Q[4] && tr > Q[8]) {
    const double s = 2.0 * std::sqrt(1.0 + tr);
    q[0] = 0.25 * s; q[1] = (Q[7] - Q[5]) / s; q[2] = (Q[2] - Q[6]) / s; q[3] = (Q[3] - Q[1]) / s;
  } else if (Q[0] > Q[4] && Q[0] > Q[8]) {
    const double s = 2.0 * std::sqrt(1.0 + Q[0] - Q[4] - Q[8]);
    q[0] = (Q[7] - Q[5]) / s; q[1] = 0.25 * s; q[2] = (Q[1] + Q[3]) / s; q[3] = (Q[2] + Q[6]) / s;
  } else if (Q[4] > Q[8]) {
    const double s = 2.0 * std::sqrt(1.0 + Q[4] - Q[0] - Q[8]);
    q[0] = (Q[2] - Q[6]) / s; q[1] = (Q[1] + Q[3]) / s; q[2] = 0.25 * s; q[3] = (Q[5] + Q[7]) / s;
  } else {
    const double s = 2.0 * std::sqrt(1.0 + Q[8] - Q[0] - Q[4]);
    q[0] = (Q[3] - Q[1]) / s; q[1] = (Q[2] + Q[6]) / s; q[2] = (Q[5] + Q[7]) / s; q[3] = 0.25 * s;
  }
  if (q[0] < 0)
    for (double& v : q) v = -v;
  const double vn = std::sqrt(q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double ang = 2.0 * std::atan2(vn, q[0]);
  for (int k = 0; k < 3; ++k) bal[k] = vn > 0 ? q[1 + k] / vn * ang : 0.0;
  double tw[3];
  mat_t_vec(R, cam + 9, tw);  // R_w2c t = R^T t
  for (int k = 0; k < 3; ++k) bal[3 + k] = -tw[k];
  bal[6] = cam[12];
  bal[7] = cam[13] / cam[12];
  bal[8] = cam[14] / cam[12];
}

// ================================================================ subproblem entry points
extern "C" int orc_camera_normal_equations(const double cam[15], int64_t n, const double* l, const double* u,
                                           const orc_options* o, double H[81], double g[9]) {
  std::vector<Coef> co((size_t)n);
  for (int64_t j = 0; j < n; ++j) co[(size_t)j] = coefficients(cam, l + 3 * j, u + 2 * j, o);
  build_normal_equations(cam, co, o, H, g);
  return 0;
}

extern "C" int orc_camera_solve(const double cam[15], int64_t n, const double* l, const double* u,
                                const orc_options* o, double out[15], int* trial, double* dP) {
  std::vector<Coef> co((size_t)n);
  for (int64_t j = 0; j < n; ++j) co[(size_t)j] = coefficients(cam, l + 3 * j, u + 2 * j, o);
  camera_lm(cam, co, u, o, out, trial, dP);
  return 0;
}

extern "C" int orc_point_solve(const double l[3], int64_t n, const double* cams, const double* u,
                               const orc_options* o, double out[3]) {
  std::vector<Coef> co((size_t)n);
  for (int64_t i = 0; i < n; ++i) co[(size_t)i] = coefficients(cams + 15 * i, l, u + 2 * i, o);
  point_closed_form(l, co, o, out);
  return 0;
}

// ================================================================ Algorithm 1
struct orc_ctx {
  int64_t M, N, K;
  orc_options o;
  std::vector<int32_t> oc, op;
  std::vector<double> uv;
  std::vector<int64_t> cam_ptr, cam_obs, pt_ptr, pt_obs;  // per-camera / per-point lists, ascending obs order
  std::vector<double> cam, cam_prev, pt, pt_prev;          // x^k, x^{k-1}
  double s = 1.0, Fbar = 0.0;                              // s^{(k)}, F-bar^{(k-1)}
  std::vector<int32_t> trial_acc, trial_mm;
  int64_t k = 0;                                           // iterations done
  // decentralized adaptive restart (§5, eqs. DEalpha, Fainit, Fak, lFak, Eak)
  int ndev = 0;                                            // 0: global restart test (D2)
  std::vector<int32_t> cam_dev, pt_dev;
  std::vector<double> dev_Fbar, dev_E;                     // F-bar^{alpha(k-1)}, E^{alpha(k)}
  std::vector<double> dev_last;                            // last iteration: ndev x ORC_DEV_COLS
};

void device_restart(orc_ctx* h, const std::vector<double>& c_acc, const std::vector<double>& c_mm,
                    const std::vector<double>& l_acc, const std::vector<double>& l_mm, std::vector<double>& cn,
                    std::vector<double>& ln, double* Fbar_sum, double* Eacc_sum, double* Emm_sum, int* n_restart);

namespace {

void build_lists(int64_t n, const std::vector<int32_t>& key, std::vector<int64_t>& ptr, std::vector<int64_t>& lst) {
  ptr.assign((size_t)n + 1, 0);
  for (int32_t k : key) ++ptr[(size_t)k + 1];
  for (int64_t i = 0; i < n; ++i) ptr[(size_t)i + 1] += ptr[(size_t)i];
  lst.resize(key.size());
  std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
  for (size_t k = 0; k < key.size(); ++k) lst[(size_t)pos[(size_t)key[k]]++] = (int64_t)k;  // stable
}

// Coefficients of camera i's observations at anchors (cams, pts).
void camera_coefs(const orc_ctx* h, int64_t i, const double* cams, const double* pts, std::vector<Coef>& co,
                  std::vector<double>& ul) {
  const int64_t b = h->cam_ptr[(size_t)i], e = h->cam_ptr[(size_t)i + 1];
  co.resize((size_t)(e - b));
  ul.resize((size_t)(2 * (e - b)));
  for (int64_t q = b; q < e; ++q) {
    const int64_t k = h->cam_obs[(size_t)q];
    const double* u = &h->uv[(size_t)(2 * k)];
    ul[(size_t)(2 * (q - b))] = u[0];
    ul[(size_t)(2 * (q - b) + 1)] = u[1];
    co[(size_t)(q - b)] = coefficients(cams + 15 * i, pts + 3 * (size_t)h->op[(size_t)k], u, &h->o);
  }
}
void point_coefs(const orc_ctx* h, int64_t j, const double* cams, const double* pts, std::vector<Coef>& co) {
  const int64_t b = h->pt_ptr[(size_t)j], e = h->pt_ptr[(size_t)j + 1];
  co.resize((size_t)(e - b));
  for (int64_t q = b; q < e; ++q) {
    const int64_t k = h->pt_obs[(size_t)q];
    co[(size_t)(q - b)] = coefficients(cams + 15 * (size_t)h->oc[(size_t)k], pts + 3 * j, &h->uv[(size_t)(2 * k)], &h->o);
  }
}

// x-bar^k (eqs. nesterov_R/t/d/l) for one camera / one point.
void extrapolate_camera(const double* c, const double* cp, double gamma, double* out) {
  double Mx[9];
  for (int k = 0; k < 9; ++k) Mx[k] = c[k] + gamma * (c[k] - cp[k]);
  orc_proj_rot3d(Mx, out);
  for (int k = 9; k < 15; ++k) out[k] = c[k] + gamma * (c[k] - cp[k]);
}
void extrapolate_point(const double* l, const double* lp, double gamma, double* out) {
  for (int k = 0; k < 3; ++k) out[k] = l[k] + gamma * (l[k] - lp[k]);
}
}  // namespace

// The two extrapolations above, exported for their pins (tests/test_oracle_iteration.py: closed-form worked values
// of eqs. nesterov_R/t/d/l).
extern "C" void orc_extrapolate_camera(const double c[15], const double cp[15], double gamma, double out[15]) {
  extrapolate_camera(c, cp, gamma, out);
}
extern "C" void orc_extrapolate_point(const double l[3], const double lp[3], double gamma, double out[3]) {
  extrapolate_point(l, lp, gamma, out);
}

namespace {

double objective(const orc_ctx* h, const double* cams, const double* pts, int64_t* ndegen) {
  // eq. Fobj: F(x) = sum over E of F_ij; degenerate pairs contribute nothing (Q17)
  Kahan tot;
  int64_t nd = 0;
  for (int64_t i = 0; i < h->M; ++i) {
    double s = 0;
    for (int64_t q = h->cam_ptr[(size_t)i]; q < h->cam_ptr[(size_t)i + 1]; ++q) {
      const int64_t k = h->cam_obs[(size_t)q];
      double F;
      if (orc_penalty(cams + 15 * i, pts + 3 * (size_t)h->op[(size_t)k], &h->uv[(size_t)(2 * k)], h->o.kind,
                      h->o.scale, h->o.eps, &F) != 0) {
        ++nd;
        continue;
      }
      s += F;
    }
    tot.add(s);
  }
  if (ndegen) *ndegen = nd;
  return tot.s;
}

}  // namespace

namespace {

// eq. DEalpha at x = x^k with anchor x^{k-1}:
//   Delta E^alpha(x^k | x^{k-1}) = -xi/2 ||x^{alpha(k)} - x^{alpha(k-1)}||^2
//     + sum_{(i,j)} kappa^alpha_ij (F_ij(c_i^k, l_j^k) - P_ij(c_i^k | x^{k-1}) - Q_ij(l_j^k | x^{k-1})).
// kappa = 1/2 for an inter-device pair touching alpha (the paper's E''_alpha).  Reading DN1: kappa = 1 for an
// intra-device pair — under D1 those pairs are majorized too, so their surrogate gap is charged wholly to their
// device (the paper keeps them exact, where the gap is 0).  With P_ij(c_hat|x_hat) = Q_ij(l_hat|x_hat) =
// F_ij(x_hat)/2 (eqs. P, Q at the anchor, by eqs. a and g) each gap is
//   F_ij(x^k) - F_ij(x^{k-1}) - dP_ij - dQ_ij    (anchor-relative changes, Q21).
std::vector<double> device_delta_E(const orc_ctx* h) {
  std::vector<Kahan> gap((size_t)h->ndev);
  for (int64_t q = 0; q < h->K; ++q) {
    const int32_t i = h->oc[(size_t)q], j = h->op[(size_t)q];
    const double* u = &h->uv[(size_t)(2 * q)];
    const Coef cp = coefficients(&h->cam_prev[(size_t)(15 * i)], &h->pt_prev[(size_t)(3 * j)], u, &h->o);
    double Fk = 0;
    if (orc_penalty(&h->cam[(size_t)(15 * i)], &h->pt[(size_t)(3 * j)], u, h->o.kind, h->o.scale, h->o.eps, &Fk) != 0)
      Fk = 0;  // Q17
    const double Fp = cp.degenerate ? 0.0 : 0.5 * cp.rho;  // eq. Fij at x^{k-1}
    const double g = Fk - Fp - pair_dP(&h->cam_prev[(size_t)(15 * i)], &h->cam[(size_t)(15 * i)], cp, u) -
                     pair_dQ(&h->pt_prev[(size_t)(3 * j)], &h->pt[(size_t)(3 * j)], cp);
    const int a = h->cam_dev[(size_t)i], b = h->pt_dev[(size_t)j];
    if (a == b) {
      gap[(size_t)a].add(g);
    } else {
      gap[(size_t)a].add(0.5 * g);
      gap[(size_t)b].add(0.5 * g);
    }
  }
  std::vector<double> dE((size_t)h->ndev);
  for (int a = 0; a < h->ndev; ++a) dE[(size_t)a] = gap[(size_t)a].s;
  for (int64_t i = 0; i < h->M; ++i) {
    double m = 0;
    for (int r = 0; r < 15; ++r) {
      const double x = h->cam[(size_t)(15 * i + r)] - h->cam_prev[(size_t)(15 * i + r)];
      m += x * x;
    }
    dE[(size_t)h->cam_dev[(size_t)i]] -= 0.5 * h->o.xi * m;
  }
  for (int64_t j = 0; j < h->N; ++j) {
    double m = 0;
    for (int r = 0; r < 3; ++r) {
      const double x = h->pt[(size_t)(3 * j + r)] - h->pt_prev[(size_t)(3 * j + r)];
      m += x * x;
    }
    dE[(size_t)h->pt_dev[(size_t)j]] -= 0.5 * h->o.xi * m;
  }
  return dE;
}

}  // namespace

// The decentralized restart of one iteration (Alg. 1 L416-420 on every device), after both candidates exist.
void device_restart(orc_ctx* h, const std::vector<double>& c_acc, const std::vector<double>& c_mm,
                    const std::vector<double>& l_acc, const std::vector<double>& l_mm, std::vector<double>& cn,
                    std::vector<double>& ln, double* Fbar_sum, double* Eacc_sum, double* Emm_sum, int* n_restart) {
  const int D = h->ndev;
  const orc_options& o = h->o;
  const std::vector<double> dE = device_delta_E(h);
  // E^alpha(x^alpha | x^k) - E^alpha(x^{alpha(k)} | x^k) of both candidates: device alpha's camera and point
  // surrogate decreases, proximal term included (eq. Ealpha restricted to alpha's variables, anchor-relative)
  std::vector<Kahan> d_acc((size_t)D), d_mm((size_t)D);
  std::vector<Coef> co;
  std::vector<double> ul;
  for (int64_t i = 0; i < h->M; ++i) {
    camera_coefs(h, i, h->cam.data(), h->pt.data(), co, ul);
    const double* ck = &h->cam[(size_t)(15 * i)];
    const size_t a = (size_t)h->cam_dev[(size_t)i];
    d_acc[a].add(camera_decrease(ck, &c_acc[(size_t)(15 * i)], co, ul.data(), &o));
    d_mm[a].add(camera_decrease(ck, &c_mm[(size_t)(15 * i)], co, ul.data(), &o));
  }
  for (int64_t j = 0; j < h->N; ++j) {
    point_coefs(h, j, h->cam.data(), h->pt.data(), co);
    const double* lk = &h->pt[(size_t)(3 * j)];
    const size_t a = (size_t)h->pt_dev[(size_t)j];
    d_acc[a].add(point_decrease(lk, &l_acc[(size_t)(3 * j)], co, &o));
    d_mm[a].add(point_decrease(lk, &l_mm[(size_t)(3 * j)], co, &o));
  }
  std::vector<char> rs((size_t)D, 0);
  Kahan fb, ea, em;
  int nrs = 0;
  h->dev_last.assign((size_t)D * ORC_DEV_COLS, 0.0);
  for (int a = 0; a < D; ++a) {
    const double F = h->dev_E[(size_t)a] + dE[(size_t)a];                    // eq. Fak
    const double Fbar = (1.0 - o.eta) * h->dev_Fbar[(size_t)a] + o.eta * F;  // eq. lFak
    const double Eacc = F + d_acc[(size_t)a].s;                              // eq. Eak, x^{alpha(k+1)} = x_acc
    const double Emm = F + d_mm[(size_t)a].s;                                // eq. Eak after a restart
    const bool r = o.accelerate ? (Eacc > Fbar) : true;                      // Alg. 1, strict ">"
    rs[(size_t)a] = r;
    nrs += (o.accelerate && r) ? 1 : 0;
    h->dev_Fbar[(size_t)a] = Fbar;
    h->dev_E[(size_t)a] = r ? Emm : Eacc;
    double* m = &h->dev_last[(size_t)a * ORC_DEV_COLS];
    m[ORC_DEV_F] = F;
    m[ORC_DEV_FBAR] = Fbar;
    m[ORC_DEV_EACC] = Eacc;
    m[ORC_DEV_EMM] = Emm;
    m[ORC_DEV_RESTART] = (o.accelerate && r) ? 1.0 : 0.0;
    fb.add(Fbar);
    ea.add(Eacc);
    em.add(Emm);
  }
  for (int64_t i = 0; i < h->M; ++i)
    std::memcpy(&cn[(size_t)(15 * i)],
                rs[(size_t)h->cam_dev[(size_t)i]] ? &c_mm[(size_t)(15 * i)] : &c_acc[(size_t)(15 * i)],
                15 * sizeof(double));
  for (int64_t j = 0; j < h->N; ++j)
    std::memcpy(&ln[(size_t)(3 * j)], rs[(size_t)h->pt_dev[(size_t)j]] ? &l_mm[(size_t)(3 * j)] : &l_acc[(size_t)(3 * j)],
                3 * sizeof(double));
  *Fbar_sum = fb.s;
  *Eacc_sum = ea.s;
  *Emm_sum = em.s;
  *n_restart = nrs;
}

extern "C" int orc_set_devices(orc_ctx* h, int ndev, const int32_t* cam_dev, const int32_t* pt_dev) {
  // Alg. 1 L403-405 with eq. Fainit: x^{alpha(-1)} = x^{alpha(0)},
  //   F^{alpha(-1)} = E^alpha(x^{alpha(-1)} | x^{(-1)}), F-bar^{alpha(-1)} = F^{alpha(-1)}, E^{alpha(0)} = F^{alpha(-1)}.
  // At its own anchor E^alpha = sum_{i in alpha} sum_j P_ij + sum_{j in alpha} sum_i Q_ij, P_ij = Q_ij = F_ij / 2.
  if (!h || ndev < 1 || !cam_dev || !pt_dev || h->k != 0) return -1;
  for (int64_t i = 0; i < h->M; ++i)
    if (cam_dev[i] < 0 || cam_dev[i] >= ndev) return -1;
  for (int64_t j = 0; j < h->N; ++j)
    if (pt_dev[j] < 0 || pt_dev[j] >= ndev) return -1;
  h->ndev = ndev;
  h->cam_dev.assign(cam_dev, cam_dev + h->M);
  h->pt_dev.assign(pt_dev, pt_dev + h->N);
  std::vector<Kahan> F0((size_t)ndev);
  for (int64_t q = 0; q < h->K; ++q) {
    const int32_t i = h->oc[(size_t)q], j = h->op[(size_t)q];
    double F = 0;
    if (orc_penalty(&h->cam[(size_t)(15 * i)], &h->pt[(size_t)(3 * j)], &h->uv[(size_t)(2 * q)], h->o.kind,
                    h->o.scale, h->o.eps, &F) != 0)
      continue;
    F0[(size_t)h->cam_dev[(size_t)i]].add(0.5 * F);  // P_ij at its anchor
    F0[(size_t)h->pt_dev[(size_t)j]].add(0.5 * F);   // Q_ij at its anchor
  }
  h->dev_Fbar.assign((size_t)ndev, 0.0);
  h->dev_E.assign((size_t)ndev, 0.0);
  for (int a = 0; a < ndev; ++a) h->dev_Fbar[(size_t)a] = h->dev_E[(size_t)a] = F0[(size_t)a].s;
  h->dev_last.assign((size_t)ndev * ORC_DEV_COLS, 0.0);
  return 0;
}

extern "C" int orc_device_metrics(const orc_ctx* h, double* out) {
  if (!h || !out || h->ndev == 0) return -1;
  std::memcpy(out, h->dev_last.data(), h->dev_last.size() * sizeof(double));
  return 0;
}

extern "C" orc_ctx* orc_create(int64_t M, const double* cams_bal, int64_t N, const double* pts, int64_t K,
                               const int32_t* obs_cam, const int32_t* obs_pt, const double* obs_uv,
                               const orc_options* o) {
  if (M < 0 || N < 0 || K < 0 || !o) return nullptr;
  orc_ctx* h = new (std::nothrow) orc_ctx();
  if (!h) return nullptr;
  h->M = M;
  h->N = N;
  h->K = K;
  h->o = *o;
  h->oc.assign(obs_cam, obs_cam + K);
  h->op.assign(obs_pt, obs_pt + K);
  h->uv.assign(obs_uv, obs_uv + 2 * K);
  for (int64_t k = 0; k < K; ++k)
    if (h->oc[(size_t)k] < 0 || h->oc[(size_t)k] >= M || h->op[(size_t)k] < 0 || h->op[(size_t)k] >= N) {
      delete h;
      return nullptr;
    }
  build_lists(M, h->oc, h->cam_ptr, h->cam_obs);
  build_lists(N, h->op, h->pt_ptr, h->pt_obs);
  h->cam.resize((size_t)(15 * M));
  for (int64_t i = 0; i < M; ++i) orc_bal_to_native(cams_bal + 9 * i, &h->cam[(size_t)(15 * i)]);
  h->pt.assign(pts, pts + 3 * N);
  // Algorithm 1: x^{(-1)} = x^{(0)}, s^{(0)} = 1, F-bar^{(-1)} = F(x^{(0)}) (eq. Fainit, global form D2)
  h->cam_prev = h->cam;
  h->pt_prev = h->pt;
  h->s = 1.0;
  h->Fbar = objective(h, h->cam.data(), h->pt.data(), nullptr);
  h->trial_acc.assign((size_t)M, -1);
  h->trial_mm.assign((size_t)M, -1);
  return h;
}

extern "C" int orc_iterate(orc_ctx* h, int n, double* trace) {
  if (!h || n < 0) return -1;
  const int64_t M = h->M, N = h->N;
  const orc_options& o = h->o;
  std::vector<double> cbar((size_t)(15 * M)), lbar((size_t)(3 * N));
  std::vector<double> c_acc((size_t)(15 * M)), c_mm((size_t)(15 * M)), l_acc((size_t)(3 * N)), l_mm((size_t)(3 * N));
  std::vector<Coef> co;
  std::vector<double> ul;
  for (int it = 0; it < n; ++it) {
    // ---- Nesterov's acceleration (Alg. 1)
    double s_next, gamma;
    orc_schedule(h->s, &s_next, &gamma);
    if (!o.accelerate) gamma = 0.0;  // DUBA ablation: plain MM
    for (int64_t i = 0; i < M; ++i)
      extrapolate_camera(&h->cam[(size_t)(15 * i)], &h->cam_prev[(size_t)(15 * i)], gamma, &cbar[(size_t)(15 * i)]);
    for (int64_t j = 0; j < N; ++j)
      extrapolate_point(&h->pt[(size_t)(3 * j)], &h->pt_prev[(size_t)(3 * j)], gamma, &lbar[(size_t)(3 * j)]);
    // (Alg. 1: with a single address space every neighbour state is already visible.)
    // ---- F(x^k) (eq. Fobj) — Lemma 1(a) makes the sum of per-device F^alpha equal to it (D2)
    int64_t ndegen = 0;
    const double Fk = objective(h, h->cam.data(), h->pt.data(), &ndegen);
    // ---- Majorization + minimization, cameras (Alg. 1; eqs. update_amm / update_mm)
    Kahan dP_acc, dP_mm, step2;
    double noacc_acc = 0, noacc_mm = 0;
    for (int64_t i = 0; i < M; ++i) {
      double dP;
      int tr;
      camera_coefs(h, i, cbar.data(), lbar.data(), co, ul);  // E(.|x-bar^k)
      camera_lm(&cbar[(size_t)(15 * i)], co, ul.data(), &o, &c_acc[(size_t)(15 * i)], &tr, &dP);
      h->trial_acc[(size_t)i] = tr;
      noacc_acc += tr < 0;
      camera_coefs(h, i, h->cam.data(), h->pt.data(), co, ul);  // E(.|x^k)
      camera_lm(&h->cam[(size_t)(15 * i)], co, ul.data(), &o, &c_mm[(size_t)(15 * i)], &tr, &dP);
      h->trial_mm[(size_t)i] = tr;
      noacc_mm += tr < 0;
      dP_mm.add(dP);
      // E(x_acc | x^k) - E(x^k | x^k), camera part (eq. Eak, global form)
      dP_acc.add(camera_decrease(&h->cam[(size_t)(15 * i)], &c_acc[(size_t)(15 * i)], co, ul.data(), &o));
    }
    // ---- points
    Kahan dQ_acc, dQ_mm;
    for (int64_t j = 0; j < N; ++j) {
      point_coefs(h, j, cbar.data(), lbar.data(), co);
      point_closed_form(&lbar[(size_t)(3 * j)], co, &o, &l_acc[(size_t)(3 * j)]);
      point_coefs(h, j, h->cam.data(), h->pt.data(), co);
      point_closed_form(&h->pt[(size_t)(3 * j)], co, &o, &l_mm[(size_t)(3 * j)]);
      dQ_acc.add(point_decrease(&h->pt[(size_t)(3 * j)], &l_acc[(size_t)(3 * j)], co, &o));
      dQ_mm.add(point_decrease(&h->pt[(size_t)(3 * j)], &l_mm[(size_t)(3 * j)], co, &o));
    }
    // ---- adaptive restart (Alg. 1; eqs. lFak, Eak in the global form D2)
    double Fbar_k = (1.0 - o.eta) * h->Fbar + o.eta * Fk;  // eq. lFak
    double E_acc = Fk + (dP_acc.s + dQ_acc.s);             // eq. Eak
    double E_mm = Fk + (dP_mm.s + dQ_mm.s);
    const bool restart = o.accelerate ? (E_acc > Fbar_k) : true;  // strict ">" (Q12)
    std::vector<double> cn = restart ? c_mm : c_acc;
    std::vector<double> ln = restart ? l_mm : l_acc;
    int n_restart = (o.accelerate && restart) ? 1 : 0;
    if (h->ndev > 0)  // decentralized: every device decides for its own variables from its local metrics
      device_restart(h, c_acc, c_mm, l_acc, l_mm, cn, ln, &Fbar_k, &E_acc, &E_mm, &n_restart);
    for (size_t q = 0; q < cn.size(); ++q) step2.add((cn[q] - h->cam[q]) * (cn[q] - h->cam[q]));
    for (size_t q = 0; q < ln.size(); ++q) step2.add((ln[q] - h->pt[q]) * (ln[q] - h->pt[q]));
    if (trace) {
      double* tr = trace + (size_t)it * ORC_TR_COLS;
      tr[ORC_TR_F] = Fk;
      tr[ORC_TR_FBAR] = Fbar_k;
      tr[ORC_TR_EACC] = E_acc;
      tr[ORC_TR_RESTART] = (double)n_restart;
      tr[ORC_TR_EMM] = E_mm;
      tr[ORC_TR_STEP2] = step2.s;
      tr[ORC_TR_GAMMA] = gamma;
      tr[ORC_TR_NDEGEN] = (double)ndegen;
      tr[ORC_TR_NOACC_ACC] = noacc_acc;
      tr[ORC_TR_NOACC_MM] = noacc_mm;
    }
    // x^{k-1} <- x^k, x^k <- x^{k+1}; s <- s^{(k+1)}; F-bar^{(k)} kept for the next iteration (Q10: no reset)
    h->cam_prev.swap(h->cam);
    h->pt_prev.swap(h->pt);
    h->cam = cn;
    h->pt = ln;
    h->s = s_next;
    h->Fbar = Fbar_k;
    ++h->k;
  }
  return 0;
}

extern "C" int orc_objective(orc_ctx* h, double* F) {
  if (!h || !F) return -1;
  *F = objective(h, h->cam.data(), h->pt.data(), nullptr);
  return 0;
}

extern "C" int orc_get_state(const orc_ctx* h, int which, double* cams, double* pts) {
  if (!h) return -1;
  const std::vector<double>& c = which ? h->cam_prev : h->cam;
  const std::vector<double>& p = which ? h->pt_prev : h->pt;
  if (cams) std::memcpy(cams, c.data(), c.size() * sizeof(double));
  if (pts) std::memcpy(pts, p.data(), p.size() * sizeof(double));
  return 0;
}

extern "C" int orc_set_state(orc_ctx* h, int which, const double* cams, const double* pts) {
  if (!h) return -1;
  std::vector<double>& c = which ? h->cam_prev : h->cam;
  std::vector<double>& p = which ? h->pt_prev : h->pt;
  if (cams) std::memcpy(c.data(), cams, c.size() * sizeof(double));
  if (pts) std::memcpy(p.data(), pts, p.size() * sizeof(double));
  return 0;
}

extern "C" int orc_set_schedule(orc_ctx* h, double s, double Fbar) {
  if (!h) return -1;
  h->s = s;
  h->Fbar = Fbar;
  return 0;
}

extern "C" int orc_get_schedule(const orc_ctx* h, double* s, double* Fbar) {
  if (!h) return -1;
  if (s) *s = h->s;
  if (Fbar) *Fbar = h->Fbar;
  return 0;
}

extern "C" int orc_last_decisions(const orc_ctx* h, int32_t* trial_acc, int32_t* trial_mm) {
  if (!h) return -1;
  if (trial_acc) std::memcpy(trial_acc, h->trial_acc.data(), h->trial_acc.size() * sizeof(int32_t));
  if (trial_mm) std::memcpy(trial_mm, h->trial_mm.data(), h->trial_mm.size() * sizeof(int32_t));
  return 0;
}

extern "C" int orc_candidates(const orc_ctx* h, int64_t ncam, const int64_t* cam_ids, double* cam_acc,
                              double* cam_mm, int64_t npt, const int64_t* pt_ids, double* pt_acc, double* pt_mm) {
  if (!h) return -1;
  double s_next, gamma;
  orc_schedule(h->s, &s_next, &gamma);
  if (!h->o.accelerate) gamma = 0.0;
  std::vector<Coef> co;
  std::vector<double> ul, lb, cb;
  for (int64_t q = 0; q < ncam; ++q) {
    const int64_t i = cam_ids[q];
    if (i < 0 || i >= h->M) return -1;
    double cbar[15];
    extrapolate_camera(&h->cam[(size_t)(15 * i)], &h->cam_prev[(size_t)(15 * i)], gamma, cbar);
    const int64_t b = h->cam_ptr[(size_t)i], e = h->cam_ptr[(size_t)i + 1];
    co.resize((size_t)(e - b));
    ul.resize((size_t)(2 * (e - b)));
    for (int64_t r = b; r < e; ++r) {
      const int64_t k = h->cam_obs[(size_t)r];
      const int64_t j = h->op[(size_t)k];
      double l[3];
      extrapolate_point(&h->pt[(size_t)(3 * j)], &h->pt_prev[(size_t)(3 * j)], gamma, l);
      ul[(size_t)(2 * (r - b))] = h->uv[(size_t)(2 * k)];
      ul[(size_t)(2 * (r - b) + 1)] = h->uv[(size_t)(2 * k + 1)];
      co[(size_t)(r - b)] = coefficients(cbar, l, &h->uv[(size_t)(2 * k)], &h->o);
    }
    int tr;
    double dP;
    camera_lm(cbar, co, ul.data(), &h->o, cam_acc + 15 * q, &tr, &dP);
    camera_coefs(h, i, h->cam.data(), h->pt.data(), co, ul);
    camera_lm(&h->cam[(size_t)(15 * i)], co, ul.data(), &h->o, cam_mm + 15 * q, &tr, &dP);
  }
  for (int64_t q = 0; q < npt; ++q) {
    const int64_t j = pt_ids[q];
    if (j < 0 || j >= h->N) return -1;
    double lbar[3];
    extrapolate_point(&h->pt[(size_t)(3 * j)], &h->pt_prev[(size_t)(3 * j)], gamma, lbar);
    const int64_t b = h->pt_ptr[(size_t)j], e = h->pt_ptr[(size_t)j + 1];
    co.resize((size_t)(e - b));
    for (int64_t r = b; r < e; ++r) {
      const int64_t k = h->pt_obs[(size_t)r];
      const int64_t i = h->oc[(size_t)k];
      double cbar[15];
      extrapolate_camera(&h->cam[(size_t)(15 * i)], &h->cam_prev[(size_t)(15 * i)], gamma, cbar);
      co[(size_t)(r - b)] = coefficients(cbar, lbar, &h->uv[(size_t)(2 * k)], &h->o);
    }
    point_closed_form(lbar, co, &h->o, pt_acc + 3 * q);
    point_coefs(h, j, h->cam.data(), h->pt.data(), co);
    point_closed_form(&h->pt[(size_t)(3 * j)], co, &h->o, pt_mm + 3 * q);
  }
  return 0;
}

extern "C" void orc_destroy(orc_ctx* h) { delete h; }
