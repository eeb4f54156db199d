"""Shared host helpers of the NEXT-3 timing tools (input preparation only; no method arithmetic)."""
import numpy as np


def bal_to_native(cams_bal):
    """BAL (angle-axis of R_w2c, t_w2c, f, k1, k2) -> native (R camera->world row-major, camera centre, (f, f k1,
    f k2)) (reading D4), vectorised numpy for timing inputs."""
    aa = np.asarray(cams_bal, np.float64).reshape(-1, 9)
    M = aa.shape[0]
    th = np.linalg.norm(aa[:, :3], axis=1, keepdims=True)
    k = aa[:, :3] / np.maximum(th, 1e-300)
    K = np.zeros((M, 3, 3))
    K[:, 0, 1], K[:, 0, 2], K[:, 1, 2] = -k[:, 2], k[:, 1], -k[:, 0]
    K = K - K.transpose(0, 2, 1)
    Rw2c = np.eye(3) + np.sin(th)[:, :, None] * K + (1 - np.cos(th))[:, :, None] * (K @ K)
    R = Rw2c.transpose(0, 2, 1)
    out = np.zeros((M, 15))
    out[:, :9] = R.reshape(-1, 9)
    out[:, 9:12] = -np.einsum("mij,mj->mi", R, aa[:, 3:6])
    out[:, 12] = aa[:, 6]
    out[:, 13] = aa[:, 6] * aa[:, 7]
    out[:, 14] = aa[:, 6] * aa[:, 8]
    return out


def camera_sorted(p):
    """(order, cam_off) putting observations in camera order."""
    order = np.argsort(p.obs_cam, kind="stable")
    off = np.concatenate([[0], np.cumsum(np.bincount(p.obs_cam, minlength=p.M))]).astype(np.int64)
    return order, off
