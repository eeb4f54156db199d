/* gen/dabagen.h — seeded synthetic bundle-adjustment problem generator.
 *
 * This module produces INPUTS only (cameras, points, observations) shaped like
 * the paper's datasets (Table 1: camera / point /
 * observation counts of BAL Ladybug, Venice, Final and 1DSfM Trafalgar).  It
 * holds none of DABA's arithmetic: no surrogate, no loss, no solver.  Both the
 * CPU oracle (oracle/) and the CUDA product path (paper_2305_07026_b200/)
 * consume its output; neither is linked into it.
 *
 * Camera model used to synthesise pixels (PAPER.md eq. reprojection1, lines
 * 102-110): the undistorted ray (u/f, 1 + k1|u|^2 + k2|u|^4) is parallel to the
 * camera-frame point R^T (l - t).  Pixels u are CENTRED coordinates (origin at
 * the principal point).  R is camera->world, t is the camera centre.
 *
 * Output camera layout is BAL 9-DoF: angle-axis of R_w2c = R^T, t_w2c = -R^T t,
 * f, k1, k2 (SURVEY.md §8(b) conventions).  Ground truth is written alongside.
 */
#ifndef DABAGEN_H
#define DABAGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { DABAGEN_SEQUENTIAL = 0, DABAGEN_CLUSTERED = 1 };

typedef struct {
  int64_t M, N, K;          /* requested cameras, points, observations (K is hit exactly when feasible) */
  int structure;            /* DABAGEN_SEQUENTIAL (street walk) or DABAGEN_CLUSTERED (photo collection rings) */
  int window;               /* sequential: candidate cameras within +-window ids of the host camera */
  int cluster_size;         /* clustered: cameras per cluster ring */
  double second_cluster_frac; /* clustered: fraction of cameras that also see a second cluster (long-range edges) */
  double noise_px;          /* Gaussian pixel noise sigma */
  double outlier_frac;      /* fraction of observations replaced by uniform-in-image pixels */
  double init_rot_deg;      /* sigma of the initial rotation perturbation (degrees, per axis) */
  double init_t_sigma;      /* sigma of the initial camera-centre perturbation (world units) */
  double init_f_frac;       /* sigma of the relative focal-length perturbation */
  double init_l_frac;       /* sigma of the point perturbation, relative to its host depth */
  int shuffle_points;       /* 1: random point-id permutation (worst-case gather locality) */
  uint64_t seed;
} dabagen_params;

void dabagen_default_params(dabagen_params* p);

/* Generate.  All output arrays are caller-owned:
 *   cams  M x 9 (BAL layout, initial state x^0)    gt_cams M x 9 (ground truth), may be NULL
 *   pts   N x 3 (initial state x^0)                gt_pts  N x 3 (ground truth), may be NULL
 *   obs_cam, obs_pt: K int32;  obs_uv: K x 2 (centred pixels)
 * Observations are emitted sorted by (camera, point).  *K_out receives the number
 * actually generated (== p->K unless the geometry could not host that many).
 * Returns 0 on success, -1 on invalid parameters. */
int dabagen_generate(const dabagen_params* p, double* cams, double* pts, int32_t* obs_cam, int32_t* obs_pt,
                     double* obs_uv, double* gt_cams, double* gt_pts, int64_t* K_out);

#ifdef __cplusplus
}
#endif
#endif
