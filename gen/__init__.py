"""Seeded synthetic DABA problems (inputs only; none of the method's arithmetic).

The generator itself is C++ (``gen/dabagen.cpp``) for speed at the Final-13682
size (29M observations); this module is its ctypes binding plus the config
table.  Shapes follow PAPER.md Table 1 (lines 508-529) and BASELINE.json's
configs; the structure recipe is SURVEY.md §8(d) "Generator v1" and DESIGN.md
"Input recipe".

Both the oracle (``oracle/``) and the CUDA product path consume these arrays;
this module imports neither.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdabagen.so")
_lib = None

SEQUENTIAL, CLUSTERED = 0, 1
LOSS_TRIVIAL, LOSS_HUBER, LOSS_CAUCHY = 0, 1, 2


class _Params(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64),
        ("structure", ctypes.c_int), ("window", ctypes.c_int), ("cluster_size", ctypes.c_int),
        ("second_cluster_frac", ctypes.c_double), ("noise_px", ctypes.c_double),
        ("outlier_frac", ctypes.c_double), ("init_rot_deg", ctypes.c_double),
        ("init_t_sigma", ctypes.c_double), ("init_f_frac", ctypes.c_double),
        ("init_l_frac", ctypes.c_double), ("shuffle_points", ctypes.c_int),
        ("seed", ctypes.c_uint64),
    ]


def build(force: bool = False) -> str:
    """Compile libdabagen.so in-tree (plain g++, no CUDA)."""
    src = os.path.join(_HERE, "dabagen.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "dabagen.h"))):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", _LIB_PATH, src])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.dabagen_default_params.argtypes = [ctypes.POINTER(_Params)]
        lib.dabagen_generate.argtypes = [ctypes.POINTER(_Params)] + [ctypes.c_void_p] * 8
        lib.dabagen_generate.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclasses.dataclass
class Problem:
    """One generated instance.  cams: M x 9 BAL (angle-axis R_w2c, t_w2c, f, k1, k2),
    pts: N x 3, obs_cam/obs_pt: K int32 sorted by (camera, point), obs_uv: K x 2 centred px."""
    name: str
    cams: np.ndarray
    pts: np.ndarray
    obs_cam: np.ndarray
    obs_pt: np.ndarray
    obs_uv: np.ndarray
    gt_cams: np.ndarray
    gt_pts: np.ndarray
    loss: int
    loss_scale: float = 1.0

    @property
    def M(self):
        return self.cams.shape[0]

    @property
    def N(self):
        return self.pts.shape[0]

    @property
    def K(self):
        return self.obs_cam.shape[0]


# name -> (M, N, K, structure, loss, outlier_frac).  Sizes from PAPER.md Table 1
# except Ladybug-49 (BAL problem-49-7776, BASELINE.json configs[0]) and the
# weak-scaling slab (BASELINE.json configs[4]).
CONFIGS = {
    "ladybug49": (49, 7776, 31843, SEQUENTIAL, LOSS_TRIVIAL, 0.0),
    "venice1778": (1778, 993923, 5001946, CLUSTERED, LOSS_HUBER, 0.03),
    "venice1778_1m": (1778, 199000, 1000000, CLUSTERED, LOSS_HUBER, 0.03),
    "trafalgar": (5032, 388956, 1826071, CLUSTERED, LOSS_HUBER, 0.03),
    "trafalgar_1m": (5032, 234000, 1100000, CLUSTERED, LOSS_HUBER, 0.03),
    "final13682": (13682, 4456117, 28987644, CLUSTERED, LOSS_HUBER, 0.03),
    "weak_slab": (14750, 4810000, 31250000, CLUSTERED, LOSS_CAUCHY, 0.03),
    # small parity cases the oracle finishes in seconds (same recipes, ragged sizes)
    "tiny_seq": (7, 61, 260, SEQUENTIAL, LOSS_TRIVIAL, 0.0),
    "small_huber": (37, 1203, 6011, CLUSTERED, LOSS_HUBER, 0.03),
    "small_cauchy": (53, 1777, 9001, CLUSTERED, LOSS_CAUCHY, 0.03),
    "small_seq_huber": (61, 2500, 11003, SEQUENTIAL, LOSS_HUBER, 0.03),
}

_SEED_BASE = 0x230507026


def generate(name: str = "ladybug49", *, seed: int | None = None, M=None, N=None, K=None,
             structure=None, loss=None, outlier_frac=None, noise_px: float = 0.5,
             init_scale: float = 1.0, shuffle_points: bool = False, cluster_size: int = 0,
             window: int = 0, loss_scale: float = 1.0) -> Problem:
    """Generate a named config (optionally overriding shape / noise).

    ``init_scale`` multiplies all initial-state perturbations (0 = start at ground
    truth).  ``noise_px=0`` and ``outlier_frac=0`` give a noiseless problem whose
    ground truth is a global minimiser (F = 0)."""
    lib = _load()
    cM, cN, cK, cs, cl, co = CONFIGS[name]
    p = _Params()
    lib.dabagen_default_params(ctypes.byref(p))
    p.M = M if M is not None else cM
    p.N = N if N is not None else cN
    p.K = K if K is not None else cK
    p.structure = structure if structure is not None else cs
    p.outlier_frac = outlier_frac if outlier_frac is not None else co
    p.noise_px = noise_px
    p.init_rot_deg *= init_scale
    p.init_t_sigma *= init_scale
    p.init_f_frac *= init_scale
    p.init_l_frac *= init_scale
    p.shuffle_points = int(shuffle_points)
    if cluster_size:
        p.cluster_size = cluster_size
    if window:
        p.window = window
    idx = list(CONFIGS).index(name)
    p.seed = (_SEED_BASE + idx) if seed is None else seed
    cams = np.empty((p.M, 9), np.float64)
    pts = np.empty((p.N, 3), np.float64)
    gt_cams = np.empty((p.M, 9), np.float64)
    gt_pts = np.empty((p.N, 3), np.float64)
    oc = np.empty(p.K, np.int32)
    op = np.empty(p.K, np.int32)
    uv = np.empty((p.K, 2), np.float64)
    kout = ctypes.c_int64(0)
    rc = lib.dabagen_generate(ctypes.byref(p), cams.ctypes.data, pts.ctypes.data, oc.ctypes.data, op.ctypes.data,
                              uv.ctypes.data, gt_cams.ctypes.data, gt_pts.ctypes.data,
                              ctypes.addressof(kout))
    if rc != 0:
        raise ValueError(f"dabagen_generate failed for {name}")
    k = kout.value
    return Problem(name, cams, pts, oc[:k].copy() if k < p.K else oc, op[:k].copy() if k < p.K else op,
                   uv[:k].copy() if k < p.K else uv, gt_cams, gt_pts,
                   loss if loss is not None else cl, loss_scale)
