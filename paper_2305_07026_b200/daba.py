"""ctypes binding of libdaba.so (include/daba.h).  Argument marshalling only: every step of the
iteration runs in the CUDA kernels behind the C-ABI; there is no CPU fallback — if the library
is missing this module raises on import of the library."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DABA_LIB", os.path.join(_HERE, "libdaba.so"))
_lib = None

LOSS_TRIVIAL, LOSS_HUBER, LOSS_CAUCHY = 0, 1, 2
COMM_NCCL, COMM_LOCAL, COMM_NONE = 0, 1, 2
(TR_F, TR_FBAR, TR_EACC, TR_RESTART, TR_EMM, TR_STEP2, TR_GAMMA, TR_NDEGEN, TR_NOACC_ACC, TR_NOACC_MM, TR_FDEV,
 TRACE_COLS) = range(12)
RESTART_GLOBAL, RESTART_DEVICE = 0, 1
ERRORS = {0: "DABA_OK", -1: "DABA_E_INVALID_ARG", -2: "DABA_E_DEGENERATE", -3: "DABA_E_CUDA", -4: "DABA_E_NCCL",
          -5: "DABA_E_OOM", -6: "DABA_E_STATE"}


class DabaError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Loss(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("scale", ctypes.c_double)]


class Options(ctypes.Structure):
    _fields_ = [("xi", ctypes.c_double), ("eta", ctypes.c_double), ("lm_mu0", ctypes.c_double),
                ("lm_mu_up", ctypes.c_double), ("eps", ctypes.c_double), ("lm_max_trials", ctypes.c_int),
                ("accelerate", ctypes.c_int), ("comm", ctypes.c_int), ("use_graph", ctypes.c_int),
                ("profile", ctypes.c_int), ("stream", ctypes.c_void_p), ("restart_scope", ctypes.c_int)]


EXPORTS = ["daba_default_options", "daba_comm_id", "daba_create", "daba_iterate", "daba_iterate_trace",
           "daba_objective", "daba_get_state", "daba_get_state_native", "daba_set_state_native",
           "daba_get_schedule", "daba_last_decisions", "daba_shard_info", "daba_stream", "daba_kernel_times",
           "daba_reset_kernel_times", "daba_launches_per_iteration", "daba_last_error", "daba_destroy",
           "daba_plan_create", "daba_plan_counts", "daba_plan_array", "daba_plan_peer_list", "daba_plan_destroy",
           "daba_pixel_error", "daba_pixel_residuals", "daba_bal_read", "daba_bal_write", "daba_bal_last_error", "daba_bal_to_paper",
           "daba_paper_to_bal", "daba_coarse_blocks", "daba_coarse_solve_workspace", "daba_coarse_solve", "daba_coarse_run",
           "daba_coarse_default_options", "daba_coarse_run_part", "daba_bal_to_native", "daba_coarse_run_dist"]


class CoarseOptions(ctypes.Structure):
    """daba_coarse_options (include/daba.h)."""
    _fields_ = [("loss", ctypes.c_int), ("scale", ctypes.c_double), ("eps", ctypes.c_double), ("xi", ctypes.c_double),
                ("eta", ctypes.c_double), ("mu0", ctypes.c_double), ("mu_up", ctypes.c_double),
                ("lm_trials", ctypes.c_int), ("accelerate", ctypes.c_int), ("pcg_max_iter", ctypes.c_int),
                ("pcg_tol", ctypes.c_double), ("mm_always", ctypes.c_int), ("keep_scratch", ctypes.c_int),
                ("deterministic", ctypes.c_int)]


def lib():
    """Load libdaba.so (built by __graft_entry__.build() / paper_2305_07026_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        V, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.daba_default_options.argtypes = [ctypes.POINTER(Options)]
        L.daba_default_options.restype = None
        L.daba_comm_id.argtypes = [V]
        L.daba_create.argtypes = [V, I64, V, I64, V, V, V, I64, Loss, V, V, I32, I32, V, I32,
                                  ctypes.POINTER(Options), ctypes.POINTER(V)]
        L.daba_iterate.argtypes = [V, I32, V, V]
        L.daba_iterate_trace.argtypes = [V, I32, V]
        L.daba_objective.argtypes = [V, ctypes.POINTER(ctypes.c_double)]
        L.daba_get_state.argtypes = [V, V, V, V]
        L.daba_get_state_native.argtypes = [V, I32, V, V, V]
        L.daba_set_state_native.argtypes = [V, V, V, V, V, ctypes.c_double, ctypes.c_double]
        L.daba_get_schedule.argtypes = [V, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(I64)]
        L.daba_last_decisions.argtypes = [V, V, V]
        L.daba_shard_info.argtypes = [V, V]
        L.daba_stream.argtypes = [V]
        L.daba_stream.restype = V
        L.daba_kernel_times.argtypes = [V, ctypes.c_char_p, ctypes.c_size_t, V, V]
        L.daba_reset_kernel_times.argtypes = [V]
        L.daba_launches_per_iteration.argtypes = [V]
        L.daba_last_error.argtypes = [V]
        L.daba_last_error.restype = ctypes.c_char_p
        L.daba_destroy.argtypes = [V]
        L.daba_destroy.restype = None
        L.daba_plan_create.argtypes = [I64, I64, V, V, I64, V, V, I32, I32]
        L.daba_plan_create.restype = V
        L.daba_plan_counts.argtypes = [V, V]
        L.daba_plan_array.argtypes = [V, I32, V]
        L.daba_plan_peer_list.argtypes = [V, I32, I32, V]
        L.daba_plan_peer_list.restype = I64
        L.daba_plan_destroy.argtypes = [V]
        L.daba_plan_destroy.restype = None
        L.daba_pixel_error.argtypes = [V, V]
        L.daba_pixel_residuals.argtypes = [V, V]
        L.daba_coarse_blocks.argtypes = [V, I64, V, I64, V, V, V, I64, I32, ctypes.c_double, ctypes.c_double, V, V, V,
                                         V, V, V, V]
        L.daba_coarse_solve_workspace.argtypes = [I64, I64]
        L.daba_coarse_solve_workspace.restype = I64
        L.daba_coarse_solve.argtypes = [V, V, V, V, V, V, V, V, I64, I64, I64, ctypes.c_double, ctypes.c_double, I32,
                                        ctypes.c_double, V, V, V, V, V]
        D = ctypes.c_double
        L.daba_coarse_run.argtypes = [V, I64, V, I64, V, V, V, V, I64, I32, D, D, D, D, D, D, I32, I32, I32, D, I32, V, V]
        L.daba_bal_to_native.argtypes = [V, I64, V]
        L.daba_coarse_run_dist.argtypes = [V, I64, V, I64, V, V, V, I64, V, V, I32, I32, V, I32, I32,
                                           ctypes.POINTER(CoarseOptions), I32, V, V, V]
        L.daba_coarse_default_options.argtypes = [ctypes.POINTER(CoarseOptions)]
        L.daba_coarse_default_options.restype = None
        L.daba_coarse_run_part.argtypes = [V, I64, V, I64, V, V, V, V, I64, V, V, I32, ctypes.POINTER(CoarseOptions),
                                           I32, V, V, V]
        L.daba_bal_read.argtypes = [ctypes.c_char_p, V, V, V, V, V, V]
        L.daba_bal_write.argtypes = [ctypes.c_char_p, V, I64, V, I64, V, V, V, I64]
        L.daba_bal_last_error.argtypes = []
        L.daba_bal_last_error.restype = ctypes.c_char_p
        L.daba_bal_to_paper.argtypes = [V, I64, V, I64]
        L.daba_paper_to_bal.argtypes = [V, I64, V, I64]
        _lib = L
    return _lib


def default_options(**kw) -> Options:
    o = Options()
    lib().daba_default_options(ctypes.byref(o))
    for k, v in kw.items():
        if k == "stream":
            v = ctypes.c_void_p(v) if v is not None else None
        setattr(o, k, v)
    return o


def comm_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().daba_comm_id(buf)
    if rc:
        raise DabaError(rc, "ncclGetUniqueId")
    return buf.raw


def _c(x, dtype):
    return np.ascontiguousarray(x, dtype=dtype)


class BalProblem:
    """A BAL dataset as arrays: cameras M x 9, points N x 3, obs_cam / obs_pt (K), obs_uv K x 2."""

    def __init__(self, cams, pts, obs_cam, obs_pt, obs_uv):
        self.cams, self.pts, self.obs_cam, self.obs_pt, self.obs_uv = cams, pts, obs_cam, obs_pt, obs_uv

    @property
    def M(self):
        return self.cams.shape[0]

    @property
    def N(self):
        return self.pts.shape[0]

    @property
    def K(self):
        return self.obs_cam.shape[0]


def read_bal(path) -> BalProblem:
    """Parse a BAL text file (daba_bal_read; native, multithreaded).  Values as written (BAL convention)."""
    L, bp = lib(), os.fsencode(path)
    counts = np.zeros(3, np.int64)
    if L.daba_bal_read(bp, counts.ctypes.data, None, None, None, None, None):
        raise DabaError(-1, L.daba_bal_last_error().decode())
    M, N, K = (int(x) for x in counts)
    cams, pts = np.empty((M, 9)), np.empty((N, 3))
    oc, op, uv = np.empty(K, np.int32), np.empty(K, np.int32), np.empty((K, 2))
    if L.daba_bal_read(bp, counts.ctypes.data, cams.ctypes.data, pts.ctypes.data, oc.ctypes.data, op.ctypes.data,
                       uv.ctypes.data):
        raise DabaError(-1, L.daba_bal_last_error().decode())
    return BalProblem(cams, pts, oc, op, uv)


def write_bal(path, prob: BalProblem) -> None:
    a = [_c(prob.cams, np.float64), _c(prob.pts, np.float64), _c(prob.obs_cam, np.int32),
         _c(prob.obs_pt, np.int32), _c(prob.obs_uv, np.float64)]
    L = lib()
    if L.daba_bal_write(os.fsencode(path), a[0].ctypes.data, a[0].shape[0], a[1].ctypes.data, a[1].shape[0],
                        a[2].ctypes.data, a[3].ctypes.data, a[4].ctypes.data, a[2].shape[0]):
        raise DabaError(-1, L.daba_bal_last_error().decode())


def _convert(fn, cams, obs_uv):
    c = np.array(cams, dtype=np.float64, order="C").reshape(-1, 9)
    u = np.array(obs_uv, dtype=np.float64, order="C").reshape(-1, 2)
    rc = fn(c.ctypes.data, c.shape[0], u.ctypes.data, u.shape[0])
    if rc:
        raise DabaError(rc, "camera with f = 0")
    return c, u


def bal_to_paper(cams, obs_uv):
    """BAL cameras / observations -> the ABI camera layout in the paper's convention (copies; daba_bal_to_paper)."""
    return _convert(lib().daba_bal_to_paper, cams, obs_uv)


def paper_to_bal(cams, obs_uv):
    """Inverse of bal_to_paper (copies; daba_paper_to_bal)."""
    return _convert(lib().daba_paper_to_bal, cams, obs_uv)


def _coarse_check(what, cams=None, pts=None, obs_cam=None, obs_pt=None, obs_uv=None, cam_off=None, extra=()):
    """Argument marshalling checks of the coarse entry points: contiguous CUDA tensors of the documented dtypes and
    shapes (the C side checks the index VALUES on the device)."""
    import torch
    f64, i32, i64 = torch.float64, torch.int32, torch.int64
    M = cams.shape[0] if cams is not None else None
    K = obs_pt.shape[0] if obs_pt is not None else None
    spec = [(cams, f64, (M, 15)), (pts, f64, (pts.shape[0], 3) if pts is not None else None),
            (obs_cam, i32, (K,)), (obs_pt, i32, (K,)), (obs_uv, f64, (K, 2)),
            (cam_off, i64, (M + 1,) if M is not None else None)] + list(extra)
    for t, dt, shape in spec:
        if t is None:
            continue
        if not (t.is_cuda and t.dtype == dt and t.is_contiguous()):
            raise DabaError(-1, f"{what}: contiguous CUDA tensors of the documented dtypes required")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise DabaError(-1, f"{what}: shape {tuple(t.shape)}, expected {tuple(shape)}")


def coarse_blocks(cams, pts, obs_pt, obs_uv, cam_off, loss=LOSS_TRIVIAL, scale=1.0, eps=1e-8, stream=None, with_W=True):
    """daba_coarse_blocks (include/daba.h): the Gauss-Newton blocks of the intra-device penalties.
    Inputs are CUDA tensors already on the device (torch: device memory only): cams (M, 15) fp64 native layout,
    pts (N, 3) fp64, obs_pt (K,) int32 and obs_uv (K, 2) fp64 sorted by camera, cam_off (M + 1,) int64.  Returns
    the CUDA tensors (U (M, 9, 9), gc (M, 9), V (N, 3, 3), gl (N, 3), W (K, 9, 3) or None when with_W is False,
    F_cam (M,)); the call is asynchronous on `stream` (default: torch's current stream)."""
    import torch
    M, N, K = cams.shape[0], pts.shape[0], obs_pt.shape[0]
    _coarse_check("coarse_blocks", cams=cams, pts=pts, obs_pt=obs_pt, obs_uv=obs_uv, cam_off=cam_off)
    dev, f64 = cams.device, torch.float64
    U, gc = torch.empty((M, 9, 9), dtype=f64, device=dev), torch.empty((M, 9), dtype=f64, device=dev)
    V, gl = torch.empty((N, 3, 3), dtype=f64, device=dev), torch.empty((N, 3), dtype=f64, device=dev)
    W = torch.empty((K, 9, 3), dtype=f64, device=dev) if with_W else None
    F = torch.empty((M,), dtype=f64, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        rc = lib().daba_coarse_blocks(cams.data_ptr(), M, pts.data_ptr(), N, obs_pt.data_ptr(), obs_uv.data_ptr(),
                                      cam_off.data_ptr(), K, int(loss), float(scale), float(eps), U.data_ptr(),
                                      gc.data_ptr(), V.data_ptr(), gl.data_ptr(), W.data_ptr() if with_W else None,
                                      F.data_ptr(), st)
    if rc != 0:
        raise DabaError(rc, "daba_coarse_blocks")
    return U, gc, V, gl, W, F


def coarse_solve(blocks, obs_cam, obs_pt, cam_off, xi=1e-4, mu=1e-3, max_iter=500, tol=1e-14, stream=None):
    """daba_coarse_solve (include/daba.h): the damped LM direction (dc (M, 9), dl (N, 3), CUDA
    tensors) of one device's coarse subproblem from coarse_blocks()' output, and (PCG iterations, residual ratio)."""
    import torch
    U, gc, V, gl, W, _ = blocks
    M, N, K = U.shape[0], V.shape[0], W.shape[0]
    f64 = torch.float64
    _coarse_check("coarse_solve", obs_cam=obs_cam, obs_pt=obs_pt,
                  extra=[(cam_off, torch.int64, (M + 1,)), (U, f64, (M, 9, 9)), (gc, f64, (M, 9)), (V, f64, (N, 3, 3)),
                         (gl, f64, (N, 3)), (W, f64, (K, 9, 3))])
    if obs_pt.shape[0] != K:
        raise DabaError(-1, "coarse_solve: obs_pt and W disagree on K")
    dev = U.device
    dc = torch.zeros((M, 9), dtype=torch.float64, device=dev)
    dl = torch.zeros((N, 3), dtype=torch.float64, device=dev)
    work = torch.empty((max(1, lib().daba_coarse_solve_workspace(M, N)),), dtype=torch.float64, device=dev)
    info = np.zeros(2)
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        rc = lib().daba_coarse_solve(U.data_ptr(), gc.data_ptr(), V.data_ptr(), gl.data_ptr(), W.data_ptr(),
                                     obs_cam.data_ptr(), obs_pt.data_ptr(), cam_off.data_ptr(), M, N, K, float(xi),
                                     float(mu), int(max_iter), float(tol), dc.data_ptr(), dl.data_ptr(), work.data_ptr(),
                                     info.ctypes.data, st)
    if rc != 0:
        raise DabaError(rc, "daba_coarse_solve")
    return dc, dl, (int(info[0]), float(info[1]))


def coarse_run(cams, pts, obs_cam, obs_pt, obs_uv, cam_off, n_iters, loss=LOSS_TRIVIAL, scale=1.0, eps=1e-8,
               xi=1e-4, eta=0.1, mu0=1e-3, mu_up=10.0, lm_trials=5, accelerate=1, pcg_max_iter=500, pcg_tol=1e-14,
               stream=None):
    """daba_coarse_run (include/daba.h; SURVEY NEXT-3 at one device): n_iters DABA iterations with the coarse
    surrogate.  cams (M, 15) / pts (N, 3) CUDA fp64 tensors are updated in place; returns the (n_iters, 5) trace."""
    import torch
    _coarse_check("coarse_run", cams=cams, pts=pts, obs_cam=obs_cam, obs_pt=obs_pt, obs_uv=obs_uv, cam_off=cam_off)
    tr = np.zeros((n_iters, 5))
    st = stream if stream is not None else torch.cuda.current_stream(cams.device).cuda_stream
    with torch.cuda.device(cams.device):
        rc = lib().daba_coarse_run(cams.data_ptr(), cams.shape[0], pts.data_ptr(), pts.shape[0], obs_cam.data_ptr(),
                                   obs_pt.data_ptr(), obs_uv.data_ptr(), cam_off.data_ptr(), obs_pt.shape[0],
                                   int(loss), float(scale), float(eps), float(xi), float(eta), float(mu0), float(mu_up),
                                   int(lm_trials), int(accelerate), int(pcg_max_iter), float(pcg_tol), int(n_iters),
                                   tr.ctypes.data, st)
    if rc != 0:
        raise DabaError(rc, "daba_coarse_run")
    return tr


def bal_to_native(cams):
    """BAL cameras (M, 9) -> the native layout (M, 15) of the coarse entry points (daba_bal_to_native)."""
    c = _c(cams, np.float64).reshape(-1, 9)
    out = np.empty((c.shape[0], 15))
    rc = lib().daba_bal_to_native(c.ctypes.data, c.shape[0], out.ctypes.data)
    if rc:
        raise DabaError(rc, "daba_bal_to_native")
    return out


def coarse_run_dist(cams, pts, obs_cam, obs_pt, obs_uv, n_iters, rank=0, nranks=1, comm_key=None, comm=COMM_NCCL,
                    device=0, cam_owner=None, pt_owner=None, **opts):
    """daba_coarse_run_dist (include/daba.h; SURVEY NEXT-3 with one device per rank): host arrays in the ABI layout
    (BAL cameras); returns (trace (n_iters, 5), cams (M, 15) native with this rank's cameras filled (NaN
    elsewhere), pts (N, 3) likewise)."""
    c, l = _c(cams, np.float64).reshape(-1, 9), _c(pts, np.float64).reshape(-1, 3)
    oc, op, uv = _c(obs_cam, np.int32), _c(obs_pt, np.int32), _c(obs_uv, np.float64).reshape(-1, 2)
    co = _c(cam_owner, np.int32) if cam_owner is not None else None
    po = _c(pt_owner, np.int32) if pt_owner is not None else None
    M, N, K = c.shape[0], l.shape[0], oc.shape[0]
    key = ctypes.create_string_buffer(comm_key, 128) if comm_key is not None else None
    o = coarse_options(**opts)
    tr = np.zeros((n_iters, 5))
    cout, lout = np.full((M, 15), np.nan), np.full((N, 3), np.nan)
    rc = lib().daba_coarse_run_dist(c.ctypes.data, M, l.ctypes.data, N, oc.ctypes.data, op.ctypes.data, uv.ctypes.data,
                                    K, co.ctypes.data if co is not None else None,
                                    po.ctypes.data if po is not None else None, rank, nranks, key, int(comm), device,
                                    ctypes.byref(o), int(n_iters), tr.ctypes.data, cout.ctypes.data, lout.ctypes.data)
    if rc != 0:
        raise DabaError(rc, "daba_coarse_run_dist")
    return tr, cout, lout


def coarse_options(**kw):
    """daba_coarse_options with the library defaults (daba_coarse_default_options) overridden by kw."""
    o = CoarseOptions()
    lib().daba_coarse_default_options(ctypes.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown coarse option {k}")
        setattr(o, k, v)
    return o


def coarse_run_part(cams, pts, obs_cam, obs_pt, obs_uv, cam_off, n_iters, cam_dev=None, pt_dev=None, ndev=None,
                    stream=None, **opts):
    """daba_coarse_run_part (include/daba.h): n_iters DABA iterations with the coarse surrogate over
    the device partition (cam_dev (M,), pt_dev (N,) int32 CUDA tensors, or None for one device).  cams / pts are
    updated in place; returns (trace (n_iters, 5), accepted trials (n_iters, 2, ndev))."""
    import torch
    M, N = cams.shape[0], pts.shape[0]
    _coarse_check("coarse_run_part", cams=cams, pts=pts, obs_cam=obs_cam, obs_pt=obs_pt, obs_uv=obs_uv,
                  cam_off=cam_off,
                  extra=[(cam_dev, torch.int32, (M,)), (pt_dev, torch.int32, (N,))])
    if (cam_dev is None) != (pt_dev is None):
        raise DabaError(-1, "coarse_run_part: cam_dev and pt_dev go together")
    if ndev is None:
        ndev = 1 if cam_dev is None else int(max(cam_dev.max().item() if M else 0, pt_dev.max().item() if N else 0)) + 1
    o = coarse_options(**opts)
    tr = np.zeros((n_iters, 5))
    trials = np.zeros((n_iters, 2, ndev), np.int32)
    st = stream if stream is not None else torch.cuda.current_stream(cams.device).cuda_stream
    with torch.cuda.device(cams.device):
        rc = lib().daba_coarse_run_part(cams.data_ptr(), M, pts.data_ptr(), N, obs_cam.data_ptr(), obs_pt.data_ptr(),
                                        obs_uv.data_ptr(), cam_off.data_ptr(), obs_pt.shape[0],
                                        cam_dev.data_ptr() if cam_dev is not None else None,
                                        pt_dev.data_ptr() if pt_dev is not None else None, int(ndev), ctypes.byref(o),
                                        int(n_iters), tr.ctypes.data, trials.ctypes.data, st)
    if rc != 0:
        raise DabaError(rc, "daba_coarse_run_part")
    return tr, trials


class Plan:
    """Host-only shard plan of one rank (the partition daba_create uses); no GPU needed."""

    def __init__(self, M, N, obs_cam, obs_pt, rank=0, nranks=1, cam_owner=None, pt_owner=None):
        oc, op = _c(obs_cam, np.int32), _c(obs_pt, np.int32)
        co = _c(cam_owner, np.int32) if cam_owner is not None else None
        po = _c(pt_owner, np.int32) if pt_owner is not None else None
        self.M, self.N = M, N
        self.h = lib().daba_plan_create(M, N, oc.ctypes.data, op.ctypes.data, oc.size,
                                        co.ctypes.data if co is not None else None,
                                        po.ctypes.data if po is not None else None, rank, nranks)
        if not self.h:
            raise DabaError(-1, "daba_plan_create")
        c = np.zeros(10, np.int64)
        lib().daba_plan_counts(self.h, c.ctypes.data)
        self.counts = dict(zip(["own_cams", "own_pts", "halo_cams", "halo_pts", "cam_side_obs", "pt_side_obs",
                                "send_doubles", "recv_doubles", "peers"], (int(v) for v in c[:9])))

    def array(self, which):
        n = {0: self.counts["own_cams"] + self.counts["halo_cams"], 1: self.counts["own_pts"] + self.counts["halo_pts"],
             2: self.M, 3: self.N, 4: self.counts["peers"]}[which]
        out = np.zeros(n, np.int32)
        lib().daba_plan_array(self.h, which, out.ctypes.data)
        return out

    def peer_list(self, peer, kind):
        n = lib().daba_plan_peer_list(self.h, peer, kind, None)
        out = np.zeros(max(n, 0), np.int32)
        lib().daba_plan_peer_list(self.h, peer, kind, out.ctypes.data)
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().daba_plan_destroy(self.h)
            self.h = None


class Solver:
    """One rank's DABA context.  Arrays follow include/daba.h (BAL cameras M x 9, points N x 3, observations
    sorted or not, pixels K x 2 centred)."""

    def __init__(self, cameras, points, obs_cam, obs_pt, obs_uv, loss=LOSS_TRIVIAL, loss_scale=1.0,
                 cam_owner=None, pt_owner=None, rank=0, nranks=1, comm_key: bytes | None = None, device=0,
                 **opts):
        L = lib()
        self._arrs = [_c(cameras, np.float64).reshape(-1, 9), _c(points, np.float64).reshape(-1, 3),
                      _c(obs_cam, np.int32), _c(obs_pt, np.int32), _c(obs_uv, np.float64).reshape(-1, 2)]
        cams, pts, oc, op, uv = self._arrs
        self.M, self.N, self.K = cams.shape[0], pts.shape[0], oc.shape[0]
        co = _c(cam_owner, np.int32) if cam_owner is not None else None
        po = _c(pt_owner, np.int32) if pt_owner is not None else None
        self.opt = default_options(**opts)
        key = ctypes.create_string_buffer(comm_key, 128) if comm_key is not None else None
        h = ctypes.c_void_p()
        rc = L.daba_create(cams.ctypes.data, self.M, pts.ctypes.data, self.N, oc.ctypes.data, op.ctypes.data,
                           uv.ctypes.data, self.K, Loss(loss, loss_scale),
                           co.ctypes.data if co is not None else None, po.ctypes.data if po is not None else None,
                           rank, nranks, key, device, ctypes.byref(self.opt), ctypes.byref(h))
        if rc:
            raise DabaError(rc, "daba_create: " + (L.daba_last_error(None) or b"").decode())
        self.h = h
        self.rank, self.nranks = rank, nranks

    def _check(self, rc, what):
        if rc < 0:
            raise DabaError(rc, f"{what}: {lib().daba_last_error(self.h).decode()}")
        return rc

    def iterate(self, n: int, F_trace: bool = False):
        """Run n iterations; returns (F(x^k) trace, restart flags) when F_trace, else None."""
        if not F_trace:
            self._check(lib().daba_iterate(self.h, n, None, None), "daba_iterate")
            return None
        F = np.zeros(n)
        r = np.zeros(n, np.uint8)
        self._check(lib().daba_iterate(self.h, n, F.ctypes.data, r.ctypes.data), "daba_iterate")
        return F, r

    def iterate_trace(self, n: int) -> np.ndarray:
        tr = np.zeros((n, TRACE_COLS))
        self._check(lib().daba_iterate_trace(self.h, n, tr.ctypes.data), "daba_iterate_trace")
        return tr

    def objective(self) -> float:
        F = ctypes.c_double()
        self._check(lib().daba_objective(self.h, ctypes.byref(F)), "daba_objective")
        return F.value

    def pixel_error(self) -> dict:
        """BAL-convention pixel reprojection error of x^k over this rank's owned cameras' observations
        (daba_pixel_error): mean, rms, number behind the camera, observations, and the raw sums."""
        out = np.zeros(4)
        self._check(lib().daba_pixel_error(self.h, out.ctypes.data), "daba_pixel_error")
        n = max(out[3], 1.0)
        return {"mean": out[0] / n, "rms": float(np.sqrt(out[1] / n)), "behind": int(out[2]), "count": int(out[3]),
                "sum": float(out[0]), "sum_sq": float(out[1])}

    def pixel_residuals(self) -> np.ndarray:
        """|r| in pixels per observation (input order) for this rank's owned cameras; NaN elsewhere
        (daba_pixel_residuals)."""
        out = np.full(self.K, np.nan)
        self._check(lib().daba_pixel_residuals(self.h, out.ctypes.data), "daba_pixel_residuals")
        return out

    def _out(self, shape):
        # entries this rank does not own stay NaN; one rank owns everything (no fill needed)
        return np.empty(shape) if self.nranks == 1 else np.full(shape, np.nan)

    def state(self):
        cams, pts = self._out((self.M, 9)), self._out((self.N, 3))
        mask = np.zeros(self.M + self.N, np.uint8)
        self._check(lib().daba_get_state(self.h, cams.ctypes.data, pts.ctypes.data, mask.ctypes.data), "get_state")
        return cams, pts, mask

    def state_native(self, which: int = 0):
        cams, pts = self._out((self.M, 15)), self._out((self.N, 3))
        mask = np.zeros(self.M + self.N, np.uint8)
        self._check(lib().daba_get_state_native(self.h, which, cams.ctypes.data, pts.ctypes.data, mask.ctypes.data),
                    "get_state_native")
        return cams, pts, mask

    def set_state_native(self, cams_k, pts_k, cams_km1, pts_km1, s, Fbar):
        a = [_c(x, np.float64) for x in (cams_k, pts_k, cams_km1, pts_km1)]
        self._check(lib().daba_set_state_native(self.h, a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data,
                                                a[3].ctypes.data, s, Fbar), "set_state_native")

    def schedule(self):
        s, Fb, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        self._check(lib().daba_get_schedule(self.h, ctypes.byref(s), ctypes.byref(Fb), ctypes.byref(k)), "schedule")
        return s.value, Fb.value, k.value

    def decisions(self):
        a, m = np.full(self.M, -2, np.int32), np.full(self.M, -2, np.int32)
        self._check(lib().daba_last_decisions(self.h, a.ctypes.data, m.ctypes.data), "decisions")
        return a, m

    def shard_info(self) -> dict:
        info = np.zeros(8, np.int64)
        self._check(lib().daba_shard_info(self.h, info.ctypes.data), "shard_info")
        keys = ["own_cams", "own_pts", "halo_cams", "halo_pts", "cam_side_obs", "pt_side_obs", "send_bytes_per_iter",
                "device_bytes"]
        return dict(zip(keys, (int(v) for v in info)))

    @property
    def stream(self) -> int:
        return lib().daba_stream(self.h) or 0

    def kernel_times(self) -> dict:
        names = ctypes.create_string_buffer(4096)
        ms = np.zeros(32)
        cnt = np.zeros(32, np.int64)
        n = self._check(lib().daba_kernel_times(self.h, names, 4096, ms.ctypes.data, cnt.ctypes.data), "kernel_times")
        keys = names.value.decode().split("\n")[:n]
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys)}

    def reset_kernel_times(self):
        self._check(lib().daba_reset_kernel_times(self.h), "reset_kernel_times")

    def launches_per_iteration(self) -> int:
        return self._check(lib().daba_launches_per_iteration(self.h), "launches_per_iteration")

    def close(self):
        if getattr(self, "h", None):
            lib().daba_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
