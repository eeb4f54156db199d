/* include/daba.h — C-ABI of the B200-native DABA hot path (libdaba.so).
 *
 * DABA = Decentralized and Accelerated Bundle Adjustment (Fan et al., arXiv 2305.07026).
 * Citations "P:L<n>" refer to the paper's LaTeX line n.
 *
 * One call of daba_iterate(ctx, n, ...) runs n iterations of Algorithm 1
 * under the readings listed in DESIGN.md: every observation is majorized by
 * Proposition 1, cameras take one successful Levenberg-Marquardt step,
 * points take the exact closed-form minimiser, Nesterov extrapolation (eqs.
 * nesterov_x0 / nesterov_x) with the adaptive restart test
 * E(x^{k+1}|x^k) > F-bar^{(k)}, evaluated either globally on one allreduced
 * vector of sums (default) or per device from the paper's local metrics
 * (DABA_RESTART_DEVICE, eqs. DEalpha-Eak).  All arithmetic is fp64 on the GPU; nothing
 * runs on the host between create and get_state.
 *
 * Conventions (all calls):
 *   - return value: 0 (DABA_OK) or a negative DABA_E_* code; daba_last_error(ctx)
 *     gives a human-readable reason for the last failure on that context;
 *   - every pointer argument is a HOST pointer unless stated otherwise; arrays are
 *     little-endian, row-major, caller-owned and copied during the call;
 *   - calls on one context are not thread-safe; distinct contexts are independent.
 *
 * Camera layouts:
 *   BAL (9 doubles):    angle-axis of R_w2c, t_w2c (3), f, k1, k2, with x_cam = R_w2c x + t_w2c.
 *   native (15 doubles): R (3x3 row-major, camera -> world), t (camera centre), d = (f, f k1, f k2);
 *                        the paper's variables: x_cam = R^T (l - t).
 *   Conversion: R = Exp(aa)^T, t = -R t_w2c, d = (f, f k1, f k2).  k1, k2 are the paper's
 *   UNDISTORTION coefficients on centred pixel coordinates (eq. reprojection1).
 */
#ifndef DABA_H
#define DABA_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define DABA_ABI_VERSION 3  /* 2: restart_scope option, DABA_TR_FDEV trace column, DABA_COMM_NONE;
                               3: BAL ingestion / conversion, daba_pixel_error */

enum {
  DABA_OK = 0,
  DABA_E_INVALID_ARG = -1, /* null/negative sizes, index out of range, duplicate (i,j), scale<=0, xi<=0, eta not in (0,1] */
  DABA_E_DEGENERATE = -2,  /* Assumption 2 fails at create: ||l_j - t_i|| <= eps for some observation */
  DABA_E_CUDA = -3,        /* CUDA runtime error (message in daba_last_error) */
  DABA_E_NCCL = -4,        /* NCCL error or unavailable library */
  DABA_E_OOM = -5,         /* device or host allocation failed */
  DABA_E_STATE = -6        /* call not valid in the context's state */
};

typedef enum { DABA_LOSS_TRIVIAL = 0, DABA_LOSS_HUBER = 1, DABA_LOSS_CAUCHY = 2 } daba_loss_kind;

/* Robust loss rho(s) of eq. Fij, s = ||e||^2; all satisfy Assumption 1.
 *   trivial: rho = s;  Huber(delta): s <= delta^2 ? s : 2 delta sqrt(s) - delta^2;
 *   Cauchy(delta): delta^2 log(1 + s / delta^2).   scale = delta > 0, in ||e|| units. */
typedef struct {
  daba_loss_kind kind;
  double scale;
} daba_loss;

enum { DABA_COMM_NCCL = 0, DABA_COMM_LOCAL = 1, DABA_COMM_NONE = 2 };

typedef struct {
  double xi;          /* proximal weight xi > 0 of eq. Ealpha; default 1e-4 */
  double eta;         /* restart averaging eta in (0,1] of eq. lFak; default 0.1 */
  double lm_mu0;      /* initial Marquardt damping; default 1e-3 */
  double lm_mu_up;    /* damping growth per failed trial; default 10 */
  double eps;         /* Assumption 2 threshold on ||l - t||; default 1e-8 */
  int lm_max_trials;  /* LM trials per camera per anchor, 1..8; default 5 */
  int accelerate;     /* 1: DABA (Nesterov + restart); 0: DUBA ablation, plain MM; default 1 */
  int comm;           /* DABA_COMM_NCCL (one process per GPU) or DABA_COMM_LOCAL (ranks = host threads of one
                         process sharing a hub; used by tests to run several ranks on one GPU); default NCCL.
                         DABA_COMM_NONE is a MEASUREMENT mode: one rank's shard runs alone, the allreduce becomes a
                         local copy and the halo exchange is skipped — the iterates are NOT the method's; it
                         times a rank's device work at nranks > 1 on one GPU (tools/shard_scaling.py). */
  int use_graph;      /* 1: capture one iteration as a CUDA graph and replay it; default 1 */
  int profile;        /* 1: record CUDA events around every kernel (see daba_kernel_times); default 0 */
  void* stream;       /* cudaStream_t to launch on (NULL: a stream owned by the context) */
  int restart_scope;  /* DABA_RESTART_GLOBAL: one restart test on the allreduced F(x^k) (reading D2, Lemma 1(a));
                         DABA_RESTART_DEVICE: the paper's decentralized scheme — every rank keeps F^{a(k)},
                         F-bar^{a(k)}, E^{a(k+1)} (eqs. DEalpha, Fainit, Fak, lFak, Eak) and decides
                         for its own cameras and points (reading DN1 in DESIGN.md).  Default GLOBAL. */
} daba_options;

enum { DABA_RESTART_GLOBAL = 0, DABA_RESTART_DEVICE = 1 };

/* Fill *o with the defaults above. */
void daba_default_options(daba_options* o);

typedef struct daba_ctx daba_ctx; /* opaque; owned by the library until daba_destroy */

/* Create a solver context on `cuda_device` for rank `rank` of `nranks`.
 *   cameras   M x 9 BAL initial cameras x^0;           points N x 3 initial points (world);
 *   obs_cam, obs_pt: K observation indices (cameras < M, points < N, each (i,j) at most once);
 *   obs_uv    K x 2 observed pixels u_ij, centred coordinates;
 *   loss      robust loss;
 *   cam_owner M ranks, or NULL: contiguous camera ranges balanced by observation count;
 *   pt_owner  N ranks, or NULL: the rank owning most of the point's observations, ties -> lowest rank;
 *   comm_id   128 bytes: an ncclUniqueId from daba_comm_id (DABA_COMM_NCCL) or any 128-byte key shared by the
 *             ranks of one DABA_COMM_LOCAL group; may be NULL iff nranks == 1 (a single rank given an id still
 *             routes its sums through the communicator);
 *   opt       options or NULL for defaults.
 * Every rank passes the same global arrays; each keeps its shard (owned cameras/points and the observations
 * touching them) plus the boundary (halo) states it reads.  Collective when nranks > 1: all ranks must call it.
 * Sets x^{-1} = x^0, s^{(0)} = 1 and F-bar^{(-1)} = F(x^0) (eq. Fainit, global form).
 * Errors: DABA_E_INVALID_ARG, DABA_E_DEGENERATE, DABA_E_CUDA, DABA_E_NCCL, DABA_E_OOM.  *out is NULL on error. */
int daba_create(const double* cameras, int64_t M, const double* points, int64_t N, const int32_t* obs_cam,
                const int32_t* obs_pt, const double* obs_uv, int64_t K, daba_loss loss, const int32_t* cam_owner,
                const int32_t* pt_owner, int rank, int nranks, const void* comm_id, int cuda_device,
                const daba_options* opt, daba_ctx** out);

/* Write a fresh 128-byte NCCL unique id into id_out (rank 0 calls this and broadcasts it).  DABA_E_NCCL if the
 * NCCL library cannot be loaded. */
int daba_comm_id(void* id_out);

/* Run n_iters iterations (collective when nranks > 1).  Optional per-iteration outputs (host, may be NULL):
 *   F_trace[k]       = F(x^k), eq. Fobj, the same on every rank;
 *   restart_trace[k] = 1 if the restart fired (x^{k+1} from eq. update_mm), else 0.
 * The call is asynchronous w.r.t. the host only when both traces are NULL and no error occurs. */
int daba_iterate(daba_ctx* ctx, int n_iters, double* F_trace, uint8_t* restart_trace);

/* Extended per-iteration trace: n_iters x DABA_TRACE_COLS doubles (host). */
/* Columns: F(x^k) (global); F-bar^{(k)}; E(x_acc|x^k); restart; E(x_mm|x^k); ||x^{k+1} - x^k||^2; gamma_k;
 * degenerate pairs (global); cameras without an accepted LM trial (acc, mm anchors; global); F^{a(k)}.
 * With DABA_RESTART_DEVICE the columns FBAR, EACC, RESTART, EMM, STEP2 and FDEV are this rank's (device a's)
 * values; with DABA_RESTART_GLOBAL they are global and FDEV = F. */
enum { DABA_TR_F = 0, DABA_TR_FBAR, DABA_TR_EACC, DABA_TR_RESTART, DABA_TR_EMM, DABA_TR_STEP2, DABA_TR_GAMMA,
       DABA_TR_NDEGEN, DABA_TR_NOACC_ACC, DABA_TR_NOACC_MM, DABA_TR_FDEV, DABA_TRACE_COLS };
int daba_iterate_trace(daba_ctx* ctx, int n_iters, double* trace);

/* F(x^k) at the current iterate (eq. Fobj), identical on every rank (collective when nranks > 1). */
int daba_objective(daba_ctx* ctx, double* F_out);

/* Current iterate x^k in BAL layout (cameras_out M x 9, points_out N x 3, either may be NULL).  Each rank writes
 * only the entries it owns; owned_mask_out (M + N bytes, nullable) receives 1 for those entries. */
int daba_get_state(daba_ctx* ctx, double* cameras_out, double* points_out, uint8_t* owned_mask_out);

/* Native-layout state.  which = 0: x^k, 1: x^{k-1}.  cameras_out M x 15, points_out N x 3 (owned entries). */
int daba_get_state_native(daba_ctx* ctx, int which, double* cameras_out, double* points_out,
                          uint8_t* owned_mask_out);

/* Overwrite x^k and x^{k-1} (native layout, GLOBAL arrays, every rank passes the same) together with the
 * schedule state s^{(k)} and F-bar^{(k-1)}: an exact resume point of Algorithm 1.  Collective. */
int daba_set_state_native(daba_ctx* ctx, const double* cams_k, const double* pts_k, const double* cams_km1,
                          const double* pts_km1, double s, double Fbar);

/* Schedule state: s^{(k)} and F-bar^{(k-1)} of the next iteration, and the iteration counter k. */
int daba_get_schedule(daba_ctx* ctx, double* s, double* Fbar, int64_t* k);

/* Accepted LM trial index per OWNED camera in the last iteration (-1: none accepted), for the accelerated and
 * the MM anchor; arrays of M int32 (global ids, non-owned entries untouched). */
int daba_last_decisions(daba_ctx* ctx, int32_t* trial_acc, int32_t* trial_mm);

/* Sizes of this rank's shard. info[0..7] = owned cams, owned points, halo cams, halo points, camera-side obs,
 * point-side obs, bytes sent per iteration, device bytes allocated. */
int daba_shard_info(daba_ctx* ctx, int64_t info[8]);

/* The cudaStream_t the context launches on (for events / synchronisation by the caller). */
void* daba_stream(daba_ctx* ctx);

/* Per-kernel device time summed since the last reset, requires opt.profile = 1.  names_out receives a
 * '\n'-separated list of kernel names (buffer of `cap` bytes), ms_out/launches_out one entry per name (up to 32).
 * Returns the number of entries (>= 0) or an error code. */
int daba_kernel_times(daba_ctx* ctx, char* names_out, size_t cap, double* ms_out, int64_t* launches_out);
int daba_reset_kernel_times(daba_ctx* ctx);

/* Number of kernel launches one iteration performs on this rank. */
int daba_launches_per_iteration(daba_ctx* ctx);

/* ---- host-only shard planning (no CUDA calls; usable on machines without a GPU) ----
 * The partition daba_create uses, exposed for tests and tooling.  Returns NULL on invalid input. */
typedef struct daba_plan daba_plan;
daba_plan* daba_plan_create(int64_t M, int64_t N, const int32_t* obs_cam, const int32_t* obs_pt, int64_t K,
                            const int32_t* cam_owner, const int32_t* pt_owner, int rank, int nranks);
/* counts[0..9] = owned cams, owned points, halo cams, halo points, camera-side obs, point-side obs, doubles sent
 * per iteration, doubles received per iteration, number of peers, (reserved 0) */
int daba_plan_counts(const daba_plan* p, int64_t counts[10]);
/* which: 0 local->global cameras (owned then halo), 1 local->global points, 2 camera owners (M), 3 point owners (N),
 *        4 peer ranks (counts[8]) */
int daba_plan_array(const daba_plan* p, int which, int32_t* out);
/* Per peer (index into the peer list): kind 0 send cameras, 1 send points, 2 recv cameras, 3 recv points, as
 * GLOBAL ids in exchange order.  Returns the length (call with out = NULL to size). */
int64_t daba_plan_peer_list(const daba_plan* p, int peer, int kind, int32_t* out);
void daba_plan_destroy(daba_plan* p);

/* Mean reprojection error in PIXELS of x^k under the BAL forward model — the accuracy metric of Table 2
 * (SURVEY NEXT-4).  For every observation of this rank's owned cameras: P' = R^T (l - t),
 * q = P'_xy / P'_z, predicted pixel f (1 + k1 |q|^2 + k2 |q|^4) q with BAL's k1 = f d2, k2 = f^3 d3 + 2 k1^2
 * (the inverse of daba_bal_to_paper's intrinsics map), residual r against the stored observation.
 * out[0] = sum |r|, out[1] = sum |r|^2, out[2] = observations with P'_z <= 0 (behind the camera; included in the
 * sums), out[3] = observations.  Mean = out[0] / out[3], RMS = sqrt(out[1] / out[3]).  Rank-local sums (the
 * caller adds them over ranks).  Runs on the device (two kernels on the context's stream), blocking. */
int daba_pixel_error(daba_ctx* ctx, double out[4]);

/* The same metric per observation: resid_out[q] = |r| (pixels) for every observation q (index into the arrays
 * given to daba_create) whose camera this rank owns; other entries are left untouched.  K doubles, host.
 * Blocking; for statistics beyond the mean (median, percentiles).  DABA_E_STATE if the context has no scratch. */
int daba_pixel_residuals(daba_ctx* ctx, double* resid_out);

/* ---- NEXT-3 building block: Gauss-Newton blocks of the coarse-partition surrogate ----
 * For a device's intra-device pairs E', whose penalties eq. Ealpha keeps exact: the blocks a
 * Schur-complement LM step on the device eliminates (readings R-N3a, R-N3b).  With the world-frame
 * residual r_k = R e (eq. error rotated; |r| = |e|), its Jacobians J_c (3x9, camera tangent (dtheta, dt, dd), left
 * rotation perturbation) and J_l (3x3), and w_k = rho'(|r_k|^2) (loss: 0 trivial, 1 Huber, 2 Cauchy; scale delta):
 *   U[i]  (81, row-major 9x9) = sum_{k of camera i} w J_c^T J_c      gc[i] (9) = sum_{k of camera i} w J_c^T r
 *   V[j]  (9, row-major 3x3)  = sum_{k of point j}  w J_l^T J_l      gl[j] (3) = sum_{k of point j}  w J_l^T r
 *   W[k]  (27, row-major 9x3) = w J_c^T J_l                          F_cam[i]  = sum_{k of camera i} rho(|r|^2)/2
 * ALL pointers are DEVICE pointers (fp64 unless stated); the caller owns every buffer.  cams: M x 15 in the native
 * layout (R camera->world row-major, t = camera centre, d = (f, f k1, f k2)); pts: N x 3; obs_pt (int32) and
 * obs_uv (K x 2) sorted by camera, with camera i's observations at [cam_off[i], cam_off[i+1]) (int64, M+1 entries).
 * W may be NULL (the per-observation blocks are then not formed: U and gc come from the structure of J_c, the
 * path daba_coarse_run takes).
 * A pair with |l - t| <= eps (Assumption 2) adds nothing and gets W[k] = 0.  V / gl are zeroed and then
 * accumulated with fp64 atomics (summation order not fixed); U / gc / F_cam are written in a fixed order.
 * The indices are checked on the device first (obs_pt in [0, N), cam_off monotone from 0 to K): DABA_E_INVALID_ARG
 * before anything is written (this synchronises `stream`).  Then asynchronous on `stream` (a cudaStream_t; NULL =
 * legacy default stream).  Returns 0, DABA_E_INVALID_ARG (-1) for bad sizes / NULL buffers / unknown loss / bad
 * indices, DABA_E_CUDA (-3) if a launch fails. */
int daba_coarse_blocks(const double* cams, int64_t M, const double* pts, int64_t N, const int32_t* obs_pt,
                       const double* obs_uv, const int64_t* cam_off, int64_t K, int loss, double scale, double eps,
                       double* U, double* gc, double* V, double* gl, double* W, double* F_cam, void* stream);

/* The damped LM direction of a device's coarse subproblem (reading R-N3c) from the blocks above:
 *   [[U + Pc, W], [W^T, V + Pl]] + mu diag(same)   [dc; dl] = -[gc; gl],
 * Pc = xi diag(2,2,2,1,1,1,1,1,1) per camera and Pl = xi I per point (the proximal term of eq. Ealpha, reading Q7).
 * Points are eliminated exactly; the reduced camera system is solved by block-Jacobi preconditioned conjugate
 * gradients (implicit Schur products, two observation passes each) until |r|_P <= tol |b|_P or max_iter
 * iterations; then dl = -(V + Pl)'^-1 (gl + W^T dc).  Inputs are daba_coarse_blocks' outputs plus obs_cam (int32,
 * sorted by camera) and the same obs_pt / cam_off; all DEVICE pointers, caller-owned.  dc: M x 9, dl: N x 3
 * (device, written).  work: daba_coarse_solve_workspace(M, N) doubles of device scratch.  The point sums W^T v use
 * fp64 atomics (reproducible to rounding); the PCG scalars are summed in a fixed order.  info (HOST, 2 doubles):
 * PCG iterations taken, final preconditioned residual ratio.  Blocking (synchronises `stream`).  Returns 0,
 * DABA_E_INVALID_ARG (-1), DABA_E_CUDA (-3), or DABA_E_STATE (-6) if a damped 3x3 / 9x9 block is not positive
 * definite (a failed LM trial: retry with a larger mu). */
int64_t daba_coarse_solve_workspace(int64_t M, int64_t N);
int daba_coarse_solve(const double* U, const double* gc, const double* V, const double* gl, const double* W,
                      const int32_t* obs_cam, const int32_t* obs_pt, const int64_t* cam_off, int64_t M, int64_t N,
                      int64_t K, double xi, double mu, int max_iter, double tol, double* dc, double* dl, double* work,
                      double info[2], void* stream);

/* Algorithm 1 with the coarse-partition surrogate on ONE device (SURVEY NEXT-3 at N = 1): every pair
 * is intra-device, so E(x | x_hat) = F(x) + xi/2 |x - x_hat|^2 (eq. Ealpha) and each of the two subproblems per
 * iteration (anchors x-bar^k and x^k, eqs. update_amm / update_mm) is one successful LM step on the whole problem
 * (readings R-N3a..d): daba_coarse_blocks, then daba_coarse_solve with mu = mu0 * mu_up^tau, tau <
 * lm_trials, accepting the first trial with a strict decrease of E.  Nesterov extrapolation with ProjRot3D and the
 * global restart test E(x_acc | x^k) > F-bar^k as in daba_iterate (reading D2; accelerate = 0: plain MM).
 * cams (M x 15 native layout) and pts (N x 3) are DEVICE buffers holding x^0 on entry and x^n on return;
 * obs_cam / obs_pt (int32), obs_uv (K x 2) DEVICE, sorted by camera with offsets cam_off (int64, M + 1, DEVICE).
 * trace (HOST, n_iters x 5, nullable): F(x^k), F-bar^k, E(x_acc | x^k), restart flag, E(x_mm | x^k).
 * Host-driven and blocking (scalars read back per LM trial); scratch is allocated stream-ordered and freed.
 * = daba_coarse_run_part with one device, mm_always = 1, keep_scratch = 1.
 * Returns 0, DABA_E_INVALID_ARG (-1), DABA_E_CUDA (-3), DABA_E_OOM (-5). */
int daba_coarse_run(double* cams, int64_t M, double* pts, int64_t N, const int32_t* obs_cam, const int32_t* obs_pt,
                    const double* obs_uv, const int64_t* cam_off, int64_t K, int loss, double scale, double eps,
                    double xi, double eta, double mu0, double mu_up, int lm_trials, int accelerate, int pcg_max_iter,
                    double pcg_tol, int n_iters, double* trace, void* stream);

/* Algorithm 1 with the coarse-partition surrogate over a DEVICE PARTITION (eq. Ealpha):
 * cam_dev (M) / pt_dev (N) give each camera / point a device in [0, ndev) (int32, DEVICE; both NULL = one device,
 * ndev = 1; ndev <= 8).  A pair whose camera and point share a device (E') is kept exactly in that device's
 * subproblem; a pair across devices (E'') is majorized (Prop. 1): P_ij on the camera's device, Q_ij on the point's.
 * Each device's subproblem (eqs. update_amm / update_mm) is one successful LM step on the device's variables
 * (readings R-N3a..d): the devices' systems are block diagonal, so one Schur-complement PCG solves them
 * all; each device accepts its first trial (mu = mu0 mu_up^tau) that strictly decreases ITS E^a, the others keep
 * trying.  The restart test is the global one of reading D2: E(x_acc | x^k) = F(x^k) + sum_a [E^a(x_acc | x^k) -
 * E^a(x^k | x^k)] > F-bar^k.  All buffers as daba_coarse_run.  trace (HOST, n_iters x 5, nullable): F(x^k),
 * F-bar^k, E(x_acc | x^k), restart flag, E(x_mm | x^k) (NaN when mm_always = 0 and no restart fired: the MM
 * subproblem is then not solved, Alg. 1).  trials (HOST, n_iters x 2 ndev int32, nullable): per iteration
 * the accepted trial of every device for the accelerated then the MM subproblem (-1: none / not solved).
 * The inputs are checked on the device first (indices in range, cam_off monotone from 0 to K, obs_cam inside its
 * camera's segment, device ids in range): DABA_E_INVALID_ARG before anything is written.  The calling thread's
 * current device is switched to the one holding `cams` for the call.  The camera-side sums and the PCG scalars are
 * taken in a fixed order; the point-side sums use fp64 atomics unless opt->deterministic (then runs are bitwise
 * reproducible).  Scratch comes from the library's stream-ordered
 * pool; keep_scratch = 0 trims the pool back afterwards.  Returns 0, DABA_E_INVALID_ARG (-1), DABA_E_CUDA (-3),
 * DABA_E_OOM (-5). */
/* The native camera layout of the coarse entry points from the ABI's BAL layout (host arrays, M x 9 -> M x 15:
 * R = Exp(aa)^T camera->world row-major, t = -R t_w2c the centre, d = (f, f k1, f k2); reading D4 — the conversion
 * daba_create applies).  0 or DABA_E_INVALID_ARG. */
int daba_bal_to_native(const double* cameras_bal, int64_t M, double* cameras_native);

typedef struct {
  int loss;          /* 0 trivial, 1 Huber, 2 Cauchy */
  double scale, eps; /* loss scale delta (> 0); Assumption 2 threshold */
  double xi, eta;    /* proximal weight (> 0), restart averaging in (0, 1] */
  double mu0, mu_up; /* LM damping schedule */
  int lm_trials;     /* >= 1 */
  int accelerate;    /* 0: plain MM (DUBA) */
  int pcg_max_iter;  /* >= 1 */
  double pcg_tol;    /* preconditioned residual ratio */
  int mm_always;     /* 1: solve the MM subproblem every iteration (oracle parity); 0: only when the restart fires */
  int keep_scratch;  /* 1: keep the scratch in the pool for the next call */
  int deterministic; /* 1: every sum in a fixed order (the point sides over a stable sort by point, made once per
                        call; no fp64 atomics): bitwise reproducible runs, ~2x slower point-side passes; 0: the
                        point-side sums by fp64 atomics (reproducible to rounding only) */
} daba_coarse_options;
void daba_coarse_default_options(daba_coarse_options* o); /* trivial, 1, 1e-8, xi 1e-4, eta 0.1, 1e-3, 10, 5, 1,
                                                              PCG <= 10 to 1e-2, mm_always 0, keep_scratch 0,
                                                              deterministic 0 */
int daba_coarse_run_part(double* cams, int64_t M, double* pts, int64_t N, const int32_t* obs_cam,
                         const int32_t* obs_pt, const double* obs_uv, const int64_t* cam_off, int64_t K,
                         const int32_t* cam_dev, const int32_t* pt_dev, int ndev, const daba_coarse_options* opt,
                         int n_iters, double* trace, int32_t* trials, void* stream);

/* The same iteration with ONE DEVICE PER RANK (SURVEY NEXT-3 distributed; the paper's setting): every rank
 * passes the same global HOST arrays (BAL cameras M x 9, points N x 3, observations as daba_create; cam_owner /
 * pt_owner: NULL = the daba_create partition) and solves its own device's subproblem on cuda_device; the halo it
 * reads (the pairs across devices) is the finest partition's; per iteration the ranks allreduce (F(x^k), the two
 * E^a decreases) and exchange the boundary variables' x^{k+1} (comm_kind 0 NCCL, 1 LOCAL threads of one process;
 * comm_id 128 bytes, NULL iff nranks == 1).  Results equal daba_coarse_run_part with cam_dev = cam_owner and
 * pt_dev = pt_owner (all devices on one GPU).  trace (HOST, n_iters x 5, same on every rank, nullable); cams_out
 * (HOST, M x 15 NATIVE layout) / pts_out (HOST, N x 3), nullable: the rank's owned entries are written.
 * Blocking.  Returns 0, DABA_E_INVALID_ARG (-1), DABA_E_CUDA (-3), DABA_E_NCCL (-4), DABA_E_OOM (-5). */
int daba_coarse_run_dist(const double* cameras, int64_t M, const double* points, int64_t N, const int32_t* obs_cam,
                         const int32_t* obs_pt, const double* obs_uv, int64_t K, const int32_t* cam_owner,
                         const int32_t* pt_owner, int rank, int nranks, const void* comm_id, int comm_kind,
                         int cuda_device, const daba_coarse_options* opt, int n_iters, double* trace,
                         double* cams_out, double* pts_out);

/* ---- BAL datasets (host only, no CUDA calls) ----
 * The BAL text format (the paper's datasets, Table 1): a header "M N K"; K observations
 * "camera point u v" (centred pixels); M cameras of 9 numbers (angle-axis of R_w2c, t_w2c, f, k1, k2 with BAL's
 * FORWARD radial distortion u = f (1 + k1 |p|^2 + k2 |p|^4) p, p = -P_xy / P_z, P = R_w2c X + t_w2c); N points
 * of 3 numbers; whitespace separated.
 *
 * daba_bal_read: with every array NULL, reads only the header into counts[3] = (M, N, K); otherwise parses the
 * whole file (multithreaded) into caller-allocated cameras (M x 9), points (N x 3), obs_cam, obs_pt (K), obs_uv
 * (K x 2), exactly as written (BAL convention).  Errors: DABA_E_INVALID_ARG — unreadable file, malformed number,
 * index out of range, too few numbers, trailing content; daba_bal_last_error() names the line (thread-local). */
int daba_bal_read(const char* path, int64_t counts[3], double* cameras, double* points, int32_t* obs_cam,
                  int32_t* obs_pt, double* obs_uv);
/* Write a BAL file (%.17g: reading it back is exact).  DABA_E_INVALID_ARG on bad arguments or an I/O error. */
int daba_bal_write(const char* path, const double* cameras, int64_t M, const double* points, int64_t N,
                   const int32_t* obs_cam, const int32_t* obs_pt, const double* obs_uv, int64_t K);
const char* daba_bal_last_error(void);
/* In place: BAL cameras (M x 9) and observations (K x 2) -> the ABI's camera layout in the paper's convention
 * (eq. reprojection1), ready for daba_create.  The paper's ray (u, f g(|u|)) must be a positive
 * multiple of R^T (l - t) while BAL's camera looks down -z: v is negated and the camera frame turned by
 * S = diag(1, -1, -1) (R^T = S R_w2c, same centre); the forward distortion is inverted by series reversion,
 * k1' = k1 / f^2, k2' = (k2 - 2 k1^2) / f^4 (exact through O(|u|^4); reading Q15).
 * DABA_E_INVALID_ARG on f = 0 or bad sizes. */
int daba_bal_to_paper(double* cameras, int64_t M, double* obs_uv, int64_t K);
/* The inverse map (round trip exact up to rounding). */
int daba_paper_to_bal(double* cameras, int64_t M, double* obs_uv, int64_t K);

/* Human-readable detail of ctx's last non-OK return; with ctx = NULL, why this thread's last daba_create failed
 * (empty if it did not).  The string is owned by the library and valid until the next call on the same ctx /
 * thread. */
const char* daba_last_error(const daba_ctx* ctx);
void daba_destroy(daba_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
