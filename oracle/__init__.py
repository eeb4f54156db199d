"""ctypes binding of the CPU oracle (oracle/daba_oracle.cpp).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs.  The product package
(paper_2305_07026_b200) never imports this module, and this module never
imports the product package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libdaba_oracle.so")
_lib = None

LOSS_TRIVIAL, LOSS_HUBER, LOSS_CAUCHY = 0, 1, 2
TR_F, TR_FBAR, TR_EACC, TR_RESTART, TR_EMM, TR_STEP2, TR_GAMMA, TR_NDEGEN, TR_NOACC_ACC, TR_NOACC_MM, TR_COLS = range(11)

_dp = ctypes.POINTER(ctypes.c_double)


class Options(ctypes.Structure):
    _fields_ = [("xi", ctypes.c_double), ("eta", ctypes.c_double), ("lm_mu0", ctypes.c_double),
                ("lm_mu_up", ctypes.c_double), ("eps", ctypes.c_double), ("lm_max_trials", ctypes.c_int),
                ("accelerate", ctypes.c_int), ("kind", ctypes.c_int), ("scale", ctypes.c_double)]


DEV_F, DEV_FBAR, DEV_EACC, DEV_EMM, DEV_RESTART, DEV_COLS = range(6)


def options(loss=LOSS_TRIVIAL, scale=1.0, xi=1e-4, eta=0.1, mu0=1e-3, mu_up=10.0, eps=1e-8, trials=5, accelerate=1):
    """Defaults are SURVEY.md D7 / DESIGN.md readings Q3, Q6, Q8, Q9."""
    return Options(xi, eta, mu0, mu_up, eps, trials, accelerate, loss, scale)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "daba_oracle.cpp")
    hdr = os.path.join(_HERE, "daba_oracle.h")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(src), os.path.getmtime(hdr)):
        # -ffp-contract=off: plain IEEE products and sums, no fused contractions.
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB, src])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        V = ctypes.c_void_p
        L.orc_create.restype = V
        L.orc_create.argtypes = [ctypes.c_int64, V, ctypes.c_int64, V, ctypes.c_int64, V, V, V, ctypes.POINTER(Options)]
        L.orc_iterate.argtypes = [V, ctypes.c_int, V]
        L.orc_objective.argtypes = [V, _dp]
        L.orc_get_state.argtypes = [V, ctypes.c_int, V, V]
        L.orc_set_state.argtypes = [V, ctypes.c_int, V, V]
        L.orc_set_schedule.argtypes = [V, ctypes.c_double, ctypes.c_double]
        L.orc_get_schedule.argtypes = [V, _dp, _dp]
        L.orc_last_decisions.argtypes = [V, V, V]
        L.orc_candidates.argtypes = [V, ctypes.c_int64, V, V, V, ctypes.c_int64, V, V, V]
        L.orc_destroy.argtypes = [V]
        L.orc_destroy.restype = None
        L.orc_set_devices.argtypes = [V, ctypes.c_int, V, V]
        L.orc_device_metrics.argtypes = [V, V]
        L.orc_ray.argtypes = [V, V, V]
        L.orc_ray.restype = None
        L.orc_optimal_scale.argtypes = [V, V, V, V, ctypes.c_double, _dp]
        L.orc_reprojection_error.argtypes = [V, V, V, V, ctypes.c_double, V]
        L.orc_loss.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp, _dp]
        L.orc_loss.restype = None
        L.orc_penalty.argtypes = [V, V, V, ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp]
        L.orc_coefficients.argtypes = [V, V, V, ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp, _dp, _dp, V]
        L.orc_P.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, V, V, V]
        L.orc_P.restype = ctypes.c_double
        L.orc_Q.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, V, V]
        L.orc_Q.restype = ctypes.c_double
        L.orc_proj_rot3d.argtypes = [V, V]
        L.orc_proj_rot3d.restype = None
        L.orc_schedule.argtypes = [ctypes.c_double, _dp, _dp]
        L.orc_schedule.restype = None
        L.orc_extrapolate_camera.argtypes = [V, V, ctypes.c_double, V]
        L.orc_extrapolate_camera.restype = None
        L.orc_extrapolate_point.argtypes = [V, V, ctypes.c_double, V]
        L.orc_extrapolate_point.restype = None
        L.orc_expmap.argtypes = [V, V]
        L.orc_expmap.restype = None
        L.orc_bal_to_native.argtypes = [V, V]
        L.orc_bal_to_native.restype = None
        L.orc_native_to_bal.argtypes = [V, V]
        L.orc_native_to_bal.restype = None
        L.orc_camera_normal_equations.argtypes = [V, ctypes.c_int64, V, V, ctypes.POINTER(Options), V, V]
        L.orc_camera_solve.argtypes = [V, ctypes.c_int64, V, V, ctypes.POINTER(Options), V,
                                       ctypes.POINTER(ctypes.c_int), _dp]
        L.orc_point_solve.argtypes = [V, ctypes.c_int64, V, V, ctypes.POINTER(Options), V]
        _lib = L
    return _lib


def _a(x, dtype=np.float64):
    return np.ascontiguousarray(x, dtype=dtype)


# ---------------------------------------------------------------- primitives
def ray(d, u):
    p = np.empty(3)
    d, u = _a(d), _a(u)
    lib().orc_ray(d.ctypes.data, u.ctypes.data, p.ctypes.data)
    return p


def optimal_scale(R, t, l, p, eps=1e-8):
    out = ctypes.c_double()
    R, t, l, p = map(_a, (R, t, l, p))
    rc = lib().orc_optimal_scale(R.ctypes.data, t.ctypes.data, l.ctypes.data, p.ctypes.data, eps, ctypes.byref(out))
    return None if rc else out.value


def reprojection_error(R, t, l, p, eps=1e-8):
    e = np.empty(3)
    R, t, l, p = map(_a, (R, t, l, p))
    rc = lib().orc_reprojection_error(R.ctypes.data, t.ctypes.data, l.ctypes.data, p.ctypes.data, eps, e.ctypes.data)
    return None if rc else e


def loss(kind, scale, s):
    r, d = ctypes.c_double(), ctypes.c_double()
    lib().orc_loss(kind, scale, s, ctypes.byref(r), ctypes.byref(d))
    return r.value, d.value


def penalty(cam15, l, u, kind=LOSS_TRIVIAL, scale=1.0, eps=1e-8):
    F = ctypes.c_double()
    cam15, l, u = map(_a, (cam15, l, u))
    rc = lib().orc_penalty(cam15.ctypes.data, l.ctypes.data, u.ctypes.data, kind, scale, eps, ctypes.byref(F))
    return None if rc else F.value


def coefficients(cam15, l, u, kind=LOSS_TRIVIAL, scale=1.0, eps=1e-8):
    a, w, lam = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    g = np.empty(3)
    cam15, l, u = map(_a, (cam15, l, u))
    rc = lib().orc_coefficients(cam15.ctypes.data, l.ctypes.data, u.ctypes.data, kind, scale, eps, ctypes.byref(a),
                                ctypes.byref(w), ctypes.byref(lam), g.ctypes.data)
    return None if rc else (a.value, w.value, lam.value, g)


def P(coef, cam15, u):
    a, w, lam, g = coef
    g, cam15, u = map(_a, (g, cam15, u))
    return lib().orc_P(a, w, lam, g.ctypes.data, cam15.ctypes.data, u.ctypes.data)


def Q(coef, l):
    a, w, lam, g = coef
    g, l = _a(g), _a(l)
    return lib().orc_Q(a, w, lam, g.ctypes.data, l.ctypes.data)


def proj_rot3d(M):
    M = _a(M).reshape(9)
    R = np.empty(9)
    lib().orc_proj_rot3d(M.ctypes.data, R.ctypes.data)
    return R.reshape(3, 3)


def schedule(s):
    sn, g = ctypes.c_double(), ctypes.c_double()
    lib().orc_schedule(s, ctypes.byref(sn), ctypes.byref(g))
    return sn.value, g.value


def extrapolate_camera(c, cp, gamma):
    """x-bar of one native camera (eqs. nesterov_R/t/d)."""
    c, cp = _a(c), _a(cp)
    out = np.empty(15)
    lib().orc_extrapolate_camera(c.ctypes.data, cp.ctypes.data, gamma, out.ctypes.data)
    return out


def extrapolate_point(l, lp, gamma):
    """x-bar of one point (eq. nesterov_l)."""
    l, lp = _a(l), _a(lp)
    out = np.empty(3)
    lib().orc_extrapolate_point(l.ctypes.data, lp.ctypes.data, gamma, out.ctypes.data)
    return out


def expmap(w):
    w = _a(w)
    R = np.empty(9)
    lib().orc_expmap(w.ctypes.data, R.ctypes.data)
    return R.reshape(3, 3)


def bal_to_native(bal):
    bal = _a(bal).reshape(-1, 9)
    out = np.empty((bal.shape[0], 15))
    for i in range(bal.shape[0]):
        lib().orc_bal_to_native(bal[i].ctypes.data, out[i].ctypes.data)
    return out


def native_to_bal(cam):
    cam = _a(cam).reshape(-1, 15)
    out = np.empty((cam.shape[0], 9))
    for i in range(cam.shape[0]):
        lib().orc_native_to_bal(cam[i].ctypes.data, out[i].ctypes.data)
    return out


def camera_normal_equations(cam15, l, u, opt):
    cam15, l, u = _a(cam15), _a(l).reshape(-1, 3), _a(u).reshape(-1, 2)
    H, g = np.empty(81), np.empty(9)
    lib().orc_camera_normal_equations(cam15.ctypes.data, l.shape[0], l.ctypes.data, u.ctypes.data, ctypes.byref(opt),
                                      H.ctypes.data, g.ctypes.data)
    return H.reshape(9, 9), g


def camera_solve(cam15, l, u, opt):
    cam15, l, u = _a(cam15), _a(l).reshape(-1, 3), _a(u).reshape(-1, 2)
    out = np.empty(15)
    tr, dP = ctypes.c_int(), ctypes.c_double()
    lib().orc_camera_solve(cam15.ctypes.data, l.shape[0], l.ctypes.data, u.ctypes.data, ctypes.byref(opt),
                           out.ctypes.data, ctypes.byref(tr), ctypes.byref(dP))
    return out, tr.value, dP.value


def point_solve(l, cams15, u, opt):
    l, cams15, u = _a(l), _a(cams15).reshape(-1, 15), _a(u).reshape(-1, 2)
    out = np.empty(3)
    lib().orc_point_solve(l.ctypes.data, cams15.shape[0], cams15.ctypes.data, u.ctypes.data, ctypes.byref(opt),
                          out.ctypes.data)
    return out


# ---------------------------------------------------------------- Algorithm 1
class Oracle:
    """Single-threaded CPU run of Algorithm 1 on a generated problem (gen.Problem)."""

    def __init__(self, prob, opt: Options | None = None, **kw):
        self.opt = opt if opt is not None else options(loss=prob.loss, scale=prob.loss_scale, **kw)
        self.M, self.N, self.K = prob.M, prob.N, prob.K
        self._keep = [_a(prob.cams), _a(prob.pts), _a(prob.obs_cam, np.int32), _a(prob.obs_pt, np.int32),
                      _a(prob.obs_uv)]
        c, p, oc, op, uv = self._keep
        self.h = lib().orc_create(self.M, c.ctypes.data, self.N, p.ctypes.data, self.K, oc.ctypes.data,
                                  op.ctypes.data, uv.ctypes.data, ctypes.byref(self.opt))
        if not self.h:
            raise ValueError("orc_create failed")

    def iterate(self, n: int) -> np.ndarray:
        tr = np.zeros((n, TR_COLS))
        if lib().orc_iterate(self.h, n, tr.ctypes.data) != 0:
            raise RuntimeError("orc_iterate failed")
        return tr

    def objective(self) -> float:
        F = ctypes.c_double()
        lib().orc_objective(self.h, ctypes.byref(F))
        return F.value

    def state(self, which: int = 0):
        cams, pts = np.empty((self.M, 15)), np.empty((self.N, 3))
        lib().orc_get_state(self.h, which, cams.ctypes.data, pts.ctypes.data)
        return cams, pts

    def set_state(self, which, cams, pts):
        cams, pts = _a(cams), _a(pts)
        lib().orc_set_state(self.h, which, cams.ctypes.data, pts.ctypes.data)

    def schedule(self):
        s, Fb = ctypes.c_double(), ctypes.c_double()
        lib().orc_get_schedule(self.h, ctypes.byref(s), ctypes.byref(Fb))
        return s.value, Fb.value

    def set_schedule(self, s, Fbar):
        lib().orc_set_schedule(self.h, s, Fbar)

    def decisions(self):
        a, m = np.empty(self.M, np.int32), np.empty(self.M, np.int32)
        lib().orc_last_decisions(self.h, a.ctypes.data, m.ctypes.data)
        return a, m

    def candidates(self, cam_ids, pt_ids):
        ci, pi = _a(cam_ids, np.int64), _a(pt_ids, np.int64)
        ca, cm = np.empty((ci.size, 15)), np.empty((ci.size, 15))
        pa, pm = np.empty((pi.size, 3)), np.empty((pi.size, 3))
        rc = lib().orc_candidates(self.h, ci.size, ci.ctypes.data, ca.ctypes.data, cm.ctypes.data, pi.size,
                                  pi.ctypes.data, pa.ctypes.data, pm.ctypes.data)
        if rc:
            raise ValueError("orc_candidates failed")
        return ca, cm, pa, pm

    def set_devices(self, cam_dev, pt_dev):
        """Decentralized adaptive restart (§5, eqs. DEalpha-Eak): device ownership of every camera and
        point; each device then takes the restart decision for its own variables.  Before the first iterate."""
        cd = np.ascontiguousarray(cam_dev, np.int32)
        pd = np.ascontiguousarray(pt_dev, np.int32)
        self.ndev = int(max(cd.max(initial=0), pd.max(initial=0))) + 1
        if lib().orc_set_devices(self.h, self.ndev, cd.ctypes.data, pd.ctypes.data) != 0:
            raise ValueError("orc_set_devices failed")

    def device_metrics(self):
        """Last iteration, per device: F^a(k), F-bar^a(k), E^a_acc(k+1), E^a_mm(k+1), restart^a."""
        out = np.zeros((self.ndev, DEV_COLS))
        if lib().orc_device_metrics(self.h, out.ctypes.data) != 0:
            raise ValueError("no device metrics")
        return out

    def close(self):
        if self.h:
            lib().orc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
