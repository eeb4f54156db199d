"""Oracle for BAL ingestion, the BAL <-> paper convention map and the pixel reprojection metric (SURVEY §8(f)
NEXT-4).  TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg,
never by the product path.  Plain numpy / scipy, no blocking or fusion; shares no code with the CUDA library.

  - parse_bal: the BAL text format as the paper's datasets ship it (Table 1; SPEC
    S:L533-551 for the field list and errors): header "M N K", K lines "camera point u v", 9 M camera numbers (angle-axis
    of R_w2c, t_w2c, f, k1, k2), 3 N point numbers.
  - bal_project: BAL's forward model, P = R_w2c X + t_w2c, p = -P_xy / P_z, u = f (1 + k1 |p|^2 + k2 |p|^4) p
    (camera looking down -z).
  - mean_pixel_error: the accuracy metric of Table 2 ("mean reprojection errors"), read as the mean
    over observations of the Euclidean pixel distance |u_obs - bal_project| (BAL projection
    convention; reading Q15).
  - bal_to_paper / paper_to_bal: the convention map of DESIGN.md reading Q15 — the paper's ray (u, f g(|u|)),
    g(s) = 1 + k1' s^2 + k2' s^4 (eq. reprojection1), must be a positive multiple of R^T (l - t):
    v -> -v, R^T = S R_w2c with S = diag(1, -1, -1), the same centre; k1' = k1 / f^2, k2' = (k2 - 2 k1^2) / f^4
    (series reversion of u = f r(|p|) p, exact through O(|u|^4)).
"""
from __future__ import annotations

import numpy as np
from scipy.spatial.transform import Rotation

S = np.diag([1.0, -1.0, -1.0])


def parse_bal(text: str):
    """BAL text -> (cams M x 9, pts N x 3, obs_cam, obs_pt, obs_uv K x 2).  ValueError on malformed input."""
    tok = text.split()
    if len(tok) < 3:
        raise ValueError("header expected")
    M, N, K = int(tok[0]), int(tok[1]), int(tok[2])
    if min(M, N, K) < 0:
        raise ValueError("negative counts")
    need = 3 + 4 * K + 9 * M + 3 * N
    if len(tok) < need:
        raise ValueError("unexpected end of file")
    if len(tok) > need:
        raise ValueError("trailing content")
    oc, op, uv = np.empty(K, np.int32), np.empty(K, np.int32), np.empty((K, 2))
    for q in range(K):
        i, j = int(tok[3 + 4 * q]), int(tok[4 + 4 * q])
        if not (0 <= i < M and 0 <= j < N):
            raise ValueError(f"observation {q}: index out of range")
        oc[q], op[q] = i, j
        uv[q] = float(tok[5 + 4 * q]), float(tok[6 + 4 * q])
    base = 3 + 4 * K
    cams = np.array([float(x) for x in tok[base:base + 9 * M]]).reshape(M, 9)
    pts = np.array([float(x) for x in tok[base + 9 * M:need]]).reshape(N, 3)
    return cams, pts, oc, op, uv


def bal_project(cam, X):
    """BAL forward projection of world points X (n x 3) by one BAL camera (9 numbers) -> pixels (n x 2)."""
    R = Rotation.from_rotvec(cam[:3]).as_matrix()
    P = np.atleast_2d(X) @ R.T + cam[3:6]
    p = -P[:, :2] / P[:, 2:3]
    n2 = np.sum(p * p, axis=1, keepdims=True)
    return cam[6] * (1.0 + cam[7] * n2 + cam[8] * n2 * n2) * p


def pixel_residuals(cams, pts, obs_cam, obs_pt, obs_uv):
    """Per observation: |u_obs - bal_project|, and whether the point is behind the BAL camera (P_z >= 0)."""
    err = np.empty(len(obs_cam))
    behind = np.zeros(len(obs_cam), bool)
    for i in np.unique(obs_cam):
        q = np.nonzero(obs_cam == i)[0]
        err[q] = np.linalg.norm(obs_uv[q] - bal_project(cams[i], pts[obs_pt[q]]), axis=1)
        R = Rotation.from_rotvec(cams[i, :3]).as_matrix()
        behind[q] = (pts[obs_pt[q]] @ R.T + cams[i, 3:6])[:, 2] >= 0.0
    return err, behind


def mean_pixel_error(cams, pts, obs_cam, obs_pt, obs_uv):
    """(sum |r|, sum |r|^2, #behind, #observations) of the BAL pixel metric (Table 2)."""
    err, behind = pixel_residuals(cams, pts, obs_cam, obs_pt, obs_uv)
    return float(err.sum()), float((err ** 2).sum()), int(behind.sum()), len(err)


def bal_to_paper(cams, obs_uv):
    """BAL cameras / pixels -> the ABI camera layout (angle-axis a' with R = Exp(a')^T, t_w2c', f, k1', k2') in the
    paper's convention, and v-flipped pixels."""
    cams = np.asarray(cams, float).reshape(-1, 9)
    out = np.empty_like(cams)
    for i, c in enumerate(cams):
        Rw = Rotation.from_rotvec(c[:3]).as_matrix()
        out[i, :3] = Rotation.from_matrix(S @ Rw).as_rotvec()
        out[i, 3:6] = S @ c[3:6]
        f, k1, k2 = c[6:9]
        out[i, 6:9] = f, k1 / f ** 2, (k2 - 2.0 * k1 ** 2) / f ** 4
    uv = np.array(obs_uv, float).reshape(-1, 2)
    uv[:, 1] = -uv[:, 1]
    return out, uv


def paper_to_bal(cams, obs_uv=None):
    """Inverse of bal_to_paper."""
    cams = np.asarray(cams, float).reshape(-1, 9)
    out = np.empty_like(cams)
    for i, c in enumerate(cams):
        Rp = Rotation.from_rotvec(c[:3]).as_matrix()
        out[i, :3] = Rotation.from_matrix(S @ Rp).as_rotvec()
        out[i, 3:6] = S @ c[3:6]
        f = c[6]
        k1 = c[7] * f ** 2
        out[i, 6:9] = f, k1, c[8] * f ** 4 + 2.0 * k1 ** 2
    if obs_uv is None:
        return out
    uv = np.array(obs_uv, float).reshape(-1, 2)
    uv[:, 1] = -uv[:, 1]
    return out, uv
