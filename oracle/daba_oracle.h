/* oracle/daba_oracle.h — single-threaded CPU oracle for one DABA iteration.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA product path (paper_2305_07026_b200/),
 * and neither includes the other.
 *
 * It implements PAPER.md (arXiv 2305.07026) Algorithm 1 (lines 394-424) under the
 * readings D1-D8 / Q1-Q23 of SURVEY.md §0 and §8(c), listed in DESIGN.md:
 *   - every observation is majorized (finest partition, D1);
 *   - one global restart test on F(x^k) computed directly (D2, Lemma 1(a));
 *   - cameras: one successful Levenberg-Marquardt step on the 9-DoF tangent,
 *     points: the exact closed-form minimiser (D3);
 *   - both surrogates (anchors x-bar^k and x^k) are built every iteration (Alg. 1).
 * Every quantity is evaluated per observation, directly from its definition.
 *
 * Native camera layout (15 doubles): R (3x3 row-major, camera -> world), t (camera
 * centre), d = (f, f k1, f k2)  — PAPER.md lines 106-110, 145-147.
 * BAL layout (9 doubles): angle-axis of R_w2c = R^T, t_w2c = -R^T t, f, k1, k2.
 *
 * Parity pins: tests/test_oracle_*.py.
 */
#ifndef DABA_ORACLE_H
#define DABA_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_LOSS_TRIVIAL = 0, ORC_LOSS_HUBER = 1, ORC_LOSS_CAUCHY = 2 };

typedef struct {
  double xi, eta, lm_mu0, lm_mu_up, eps;
  int lm_max_trials, accelerate;
  int kind;     /* robust loss kind */
  double scale; /* robust loss scale delta (in ||e|| units) */
} orc_options;

/* ---- geometry (§3) ---- */
void orc_ray(const double d[3], const double u[2], double p[3]);                        /* eq. ray */
int orc_optimal_scale(const double R[9], const double t[3], const double l[3], const double p[3], double eps,
                      double* lambda);                                                    /* eq. lambdaij */
int orc_reprojection_error(const double R[9], const double t[3], const double l[3], const double p[3], double eps,
                           double e[3]);                                                  /* eq. error */
void orc_loss(int kind, double scale, double s, double* rho, double* drho);              /* Assumption 1 */
int orc_penalty(const double cam[15], const double l[3], const double u[2], int kind, double scale, double eps,
                double* F);                                                               /* eq. Fij */
/* ---- surrogate (§4, Prop. 1) ---- */
int orc_coefficients(const double cam[15], const double l[3], const double u[2], int kind, double scale, double eps,
                     double* a, double* w, double* lambda, double g[3]);                  /* eqs. a, w, gamma, g */
double orc_P(double a, double w, double lambda, const double g[3], const double cam[15], const double u[2]); /* eq. P */
double orc_Q(double a, double w, double lambda, const double g[3], const double l[3]);                        /* eq. Q */
/* ---- acceleration (§5) ---- */
void orc_proj_rot3d(const double M[9], double R[9]);                                       /* eq. proj_rot3d */
void orc_schedule(double s, double* s_next, double* gamma);                                /* eq. nesterov_scalar */
/* x-bar from x^k (c, l) and x^{k-1} (cp, lp): eqs. nesterov_R/t/d (ProjRot3D of the extrapolated R) and
 * nesterov_l */
void orc_extrapolate_camera(const double c[15], const double cp[15], double gamma, double out[15]);
void orc_extrapolate_point(const double l[3], const double lp[3], double gamma, double out[3]);
void orc_expmap(const double w[3], double R[9]);
void orc_bal_to_native(const double bal[9], double cam[15]);
void orc_native_to_bal(const double cam[15], double bal[9]);
/* ---- subproblem solvers (D3) ---- */
/* Camera subproblem at anchor `cam` over `n` observations with anchor points l (n x 3), pixels u (n x 2),
 * anchor cameras are `cam` for all of them.  H (81) and g (9) are the Gauss-Newton normal equations of
 * sum_j P_j(c) + xi/2 ||c - c_hat||^2 on the tangent (dtheta, dt, dd) at the anchor. */
int orc_camera_normal_equations(const double cam[15], int64_t n, const double* l, const double* u,
                                const orc_options* o, double H[81], double g[9]);
/* One successful LM step (<= lm_max_trials trials).  out: 15 doubles; *trial = accepted trial index or -1;
 * *dP = surrogate decrease of the accepted trial (0 if none). */
int orc_camera_solve(const double cam[15], int64_t n, const double* l, const double* u, const orc_options* o,
                     double out[15], int* trial, double* dP);
/* Exact point minimiser of sum_i Q_ij(l) + xi/2 ||l - l_hat||^2; cams: n x 15 anchor cameras. */
int orc_point_solve(const double l[3], int64_t n, const double* cams, const double* u, const orc_options* o,
                    double out[3]);

/* ---- the iteration (Algorithm 1) ---- */
typedef struct orc_ctx orc_ctx;
/* trace columns per iteration k */
enum { ORC_TR_F = 0, ORC_TR_FBAR, ORC_TR_EACC, ORC_TR_RESTART, ORC_TR_EMM, ORC_TR_STEP2, ORC_TR_GAMMA, ORC_TR_NDEGEN,
       ORC_TR_NOACC_ACC, ORC_TR_NOACC_MM, ORC_TR_COLS };
orc_ctx* orc_create(int64_t M, const double* cams_bal, int64_t N, const double* pts, int64_t K,
                    const int32_t* obs_cam, const int32_t* obs_pt, const double* obs_uv, const orc_options* o);
int orc_iterate(orc_ctx* h, int n, double* trace /* n x ORC_TR_COLS, nullable */);
int orc_objective(orc_ctx* h, double* F);
/* which: 0 = x^k, 1 = x^{k-1}; cams: M x 15 native, pts: N x 3 */
int orc_get_state(const orc_ctx* h, int which, double* cams, double* pts);
int orc_set_state(orc_ctx* h, int which, const double* cams, const double* pts);
int orc_set_schedule(orc_ctx* h, double s, double Fbar);
int orc_get_schedule(const orc_ctx* h, double* s, double* Fbar);
/* accepted LM trial per camera in the last iteration (acc and mm anchors), M each */
int orc_last_decisions(const orc_ctx* h, int32_t* trial_acc, int32_t* trial_mm);
/* Sampled single-iteration candidates from the current (x^k, x^{k-1}, s): for the listed cameras
 * and points, the accelerated (x-bar anchored) and MM (x^k anchored) solutions. */
int orc_candidates(const orc_ctx* h, int64_t ncam, const int64_t* cam_ids, double* cam_acc, double* cam_mm,
                   int64_t npt, const int64_t* pt_ids, double* pt_acc, double* pt_mm);
/* Decentralized adaptive restart (§5, eqs. DEalpha, Fainit, Fak, lFak, Eak; Alg. 1): from
 * now on every device alpha (cam_dev: M entries, pt_dev: N entries, in [0, ndev)) keeps F^{alpha(k)},
 * F-bar^{alpha(k)}, E^{alpha(k+1)} and takes the restart decision for its own variables.  Must be called
 * before the first iteration.  The trace then holds F(x^k) in ORC_TR_F, sums over devices in FBAR / EACC /
 * EMM and the number of restarting devices in RESTART. */
enum { ORC_DEV_F = 0, ORC_DEV_FBAR, ORC_DEV_EACC, ORC_DEV_EMM, ORC_DEV_RESTART, ORC_DEV_COLS };
int orc_set_devices(orc_ctx* h, int ndev, const int32_t* cam_dev, const int32_t* pt_dev);
/* last iteration's per-device metrics, ndev x ORC_DEV_COLS */
int orc_device_metrics(const orc_ctx* h, double* out);
void orc_destroy(orc_ctx* h);

#ifdef __cplusplus
}
#endif
#endif
