"""Shared host helpers of the NEXT-3 timing tools (input preparation only; no method arithmetic)."""
import numpy as np

import paper_2305_07026_b200 as daba


def bal_to_native(cams_bal):
    """BAL cameras -> the native layout of the coarse entry points, by the library's own conversion
    (daba_bal_to_native, reading D4)."""
    return daba.bal_to_native(cams_bal)


def camera_sorted(p):
    """(order, cam_off) putting observations in camera order."""
    order = np.argsort(p.obs_cam, kind="stable")
    off = np.concatenate([[0], np.cumsum(np.bincount(p.obs_cam, minlength=p.M))]).astype(np.int64)
    return order, off


def contiguous_partition(p, ndev):
    """Cameras in ndev contiguous id ranges balanced by observation count, each point on the device owning
    most of its observations (ties: lowest) — the engine's planner (shard.h), for the coarse timing tools."""
    cnt = np.bincount(p.obs_cam, minlength=p.M)
    cum = np.cumsum(cnt) - cnt
    cam_dev = np.minimum(cum * ndev // max(p.K, 1), ndev - 1).astype(np.int32)
    votes = np.zeros((p.N, ndev), np.int64)
    np.add.at(votes, (p.obs_pt, cam_dev[p.obs_cam]), 1)
    return cam_dev, votes.argmax(axis=1).astype(np.int32)
