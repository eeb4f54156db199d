"""NEXT-3 oracle: DABA with the paper's coarse-partition surrogate.

TEST INFRASTRUCTURE ONLY: importable from tests/ (and nothing else).  It never imports the product package
(paper_2305_07026_b200); the geometry primitives it calls (ray, optimal scale, loss, penalty, coefficients,
eqs. P / Q, the camera normal equations of the majorized pairs, Exp, ProjRot3D, the schedule) are the C
oracle's, pinned by tests/test_oracle_geometry.py and tests/test_oracle_surrogate.py.

What it computes (PAPER.md, arXiv 2305.07026):
  - the split of the reprojection pairs into E' (camera and point on the same device) and E'' (different
    devices);
  - the device surrogate E^a(x^a | x_hat) of eq. Ealpha: the intra-device penalties F_ij kept
    exactly, the inter-device pairs majorized by P_ij (camera side, on the camera's device) and Q_ij (point side,
    on the point's device) of Prop. 1 (eqs. P, Q), plus xi/2 ||x^a - x_hat^a||^2;
  - each device subproblem (eqs. update_amm / update_mm) approximated by ONE successful
    Levenberg-Marquardt step on the device's stacked tangent (9 per camera, 3 per point) -- reading
    R-N3a..R-N3d of DESIGN.md §2;
  - Algorithm 1 with the global restart test of reading D2: E(x_acc^{k+1} | x^k) > F-bar^k.

Readings ("NEXT-3"):
  R-N3a  F_ij in E' enters the LM normal equations by Gauss-Newton with the robust weight w = rho'(|e|^2)
         (H += w J^T J, g += w J^T e); the trial is accepted on the exact surrogate decrease.
  R-N3b  residual e in the world frame: R e = Pi_v R p with v = l - t and Pi_v = I - v v^T / |v|^2 (eq. error
         rotated by R, |R e| = |e|); Jacobians derived below and pinned by central differences.
  R-N3c  damping, trials and Jacobi scaling as the camera LM of reading D3: Marquardt H + mu diag(H),
         mu = mu0 * mu_up^tau, first strict decrease accepted, else the anchor is kept.
  R-N3d  a pair that is degenerate (Assumption 2, |l - t| <= eps) at the anchor contributes nothing to the
         normal equations; F_ij of a degenerate pair is 0 in every evaluation (reading Q17).
"""
from __future__ import annotations

import numpy as np

from . import (bal_to_native, camera_normal_equations, coefficients, expmap, loss, optimal_scale, options, P, penalty,
               Q, proj_rot3d, ray, schedule)


def skew(a):
    return np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])


# ---------------------------------------------------------------- one pair: residual and Jacobians (R-N3b)
def residual(cam, l, u, eps=1e-8):
    """World-frame reprojection error R e (eq. error, rotated by R) or None (Assumption 2)."""
    R, t = cam[:9].reshape(3, 3), cam[9:12]
    p = ray(cam[12:15], u)
    lam = optimal_scale(R, t, l, p, eps)  # eq. lambdaij
    if lam is None:
        return None
    return R @ p - lam * (l - t)


def residual_jacobians(cam, l, u, eps=1e-8):
    """(r, J_c 3x9, J_l 3x3) of r = R e at (cam, l): camera tangent (dtheta, dt, dd) with the left perturbation
    R = Exp(dtheta) R_hat (reading Q5), point tangent dl.  With q = R p(d), v = l - t, lam = v.q / |v|^2:
      dr/dq = Pi_v,  dr/dv = -(v q^T) / |v|^2 - lam I + 2 lam v v^T / |v|^2,
      dq/dtheta = -[q]_x,  dq/dd = R e_3 b^T with b = (1, |u|^2, |u|^4) (eq. ray),  dv/dt = -I,  dv/dl = I."""
    R, t = cam[:9].reshape(3, 3), cam[9:12]
    p = ray(cam[12:15], u)
    lam = optimal_scale(R, t, l, p, eps)
    if lam is None:
        return None
    q = R @ p
    v = l - t
    nv = v @ v
    Pi = np.eye(3) - np.outer(v, v) / nv
    Dv = -np.outer(v, q) / nv - lam * np.eye(3) + 2.0 * lam * np.outer(v, v) / nv
    s = u @ u
    b = np.array([1.0, s, s * s])
    Jc = np.zeros((3, 9))
    Jc[:, 0:3] = Pi @ (-skew(q))
    Jc[:, 3:6] = -Dv
    Jc[:, 6:9] = Pi @ np.outer(R[:, 2], b)
    return q - lam * v, Jc, Dv


def retract_camera(cam, delta):
    """c' = (Exp(dtheta) R_hat, t + dt, d + dd) (reading Q5)."""
    out = np.array(cam, dtype=np.float64)
    out[:9] = (expmap(delta[0:3]) @ cam[:9].reshape(3, 3)).reshape(9)
    out[9:12] = cam[9:12] + delta[3:6]
    out[12:15] = cam[12:15] + delta[6:9]
    return out


# ---------------------------------------------------------------- problem and partition
class Problem:
    """Native-layout copy of a generated problem (gen.Problem) with a device assignment of cameras and points."""

    def __init__(self, prob, cam_dev, pt_dev, opt=None, **kw):
        self.opt = opt if opt is not None else options(loss=prob.loss, scale=prob.loss_scale, **kw)
        self.M, self.N, self.K = prob.M, prob.N, prob.K
        self.cams0 = np.asarray(bal_to_native(np.asarray(prob.cams, np.float64)), np.float64).reshape(-1, 15).copy()
        self.pts0 = np.asarray(prob.pts, np.float64).reshape(-1, 3).copy()
        self.oc = np.asarray(prob.obs_cam, np.int64)
        self.op = np.asarray(prob.obs_pt, np.int64)
        self.uv = np.asarray(prob.obs_uv, np.float64).reshape(-1, 2)
        self.cam_dev = np.asarray(cam_dev, np.int64)
        self.pt_dev = np.asarray(pt_dev, np.int64)
        self.devices = sorted(set(self.cam_dev.tolist()) | set(self.pt_dev.tolist()))
        self.intra = self.cam_dev[self.oc] == self.pt_dev[self.op]  # E'
        # pairs whose camera or point lives on device a (the only terms of E^a)
        self.touch = {a: np.flatnonzero((self.cam_dev[self.oc] == a) | (self.pt_dev[self.op] == a))
                      for a in self.devices}
        self.cam_pairs = [[] for _ in range(self.M)]
        for k in range(self.K):
            self.cam_pairs[self.oc[k]].append(k)

    # eq. Fobj
    def F_pair(self, k, cams, pts):
        o = self.opt
        f = penalty(cams[self.oc[k]], pts[self.op[k]], self.uv[k], o.kind, o.scale, o.eps)
        return 0.0 if f is None else f

    def objective(self, cams, pts):
        return float(sum(self.F_pair(k, cams, pts) for k in range(self.K)))

    def coef(self, k, cams_hat, pts_hat):
        o = self.opt
        return coefficients(cams_hat[self.oc[k]], pts_hat[self.op[k]], self.uv[k], o.kind, o.scale, o.eps)

    # eq. Ealpha, every device summed: E(x | x_hat)
    def surrogate(self, cams, pts, cams_hat, pts_hat, devices=None):
        """sum over the listed devices (default: all) of E^a(x^a | x_hat)."""
        devs = set(self.devices if devices is None else devices)
        tot = 0.0
        ks = range(self.K) if devices is None else sorted(set().union(*(self.touch[a].tolist() for a in devs)))
        for k in ks:
            i, j = self.oc[k], self.op[k]
            ci, pj = self.cam_dev[i] in devs, self.pt_dev[j] in devs
            if self.intra[k]:
                if ci:
                    tot += self.F_pair(k, cams, pts)
                continue
            c = self.coef(k, cams_hat, pts_hat)
            if c is None:  # R-N3d
                continue
            if ci:
                tot += P(c, cams[i], self.uv[k])
            if pj:
                tot += Q(c, pts[j])
        cm = np.isin(self.cam_dev, list(devs))
        pm = np.isin(self.pt_dev, list(devs))
        prox = np.sum((cams - cams_hat)[cm] ** 2) + np.sum((pts - pts_hat)[pm] ** 2)
        return tot + 0.5 * self.opt.xi * prox

    # ------------------------------------------------------------ one device subproblem, one successful LM step
    def device_system(self, a, cams_hat, pts_hat):
        """Gauss-Newton normal equations (H, g) of E^a(. | x_hat) at x_hat^a on the device's stacked tangent (9 per
        camera in ascending id, then 3 per point), proximal term included (R-N3a); also the variable layout."""
        o = self.opt
        ci = np.flatnonzero(self.cam_dev == a)
        pj = np.flatnonzero(self.pt_dev == a)
        cpos = {int(i): 9 * n for n, i in enumerate(ci)}
        ppos = {int(j): 9 * len(ci) + 3 * n for n, j in enumerate(pj)}
        n = 9 * len(ci) + 3 * len(pj)
        H = np.zeros((n, n))
        g = np.zeros(n)
        # inter-device camera side: the C oracle's majorized normal equations (eq. P, with the camera's prox)
        for i in ci:
            ks = [k for k in self.cam_pairs[i] if not self.intra[k]]
            Hc, gc = camera_normal_equations(cams_hat[i], pts_hat[self.op[ks]].reshape(-1, 3),
                                             self.uv[ks].reshape(-1, 2), o)
            s = cpos[int(i)]
            H[s:s + 9, s:s + 9] += Hc
            g[s:s + 9] += gc
        for j in pj:
            s = ppos[int(j)]
            H[s:s + 3, s:s + 3] += o.xi * np.eye(3)  # eq. Ealpha prox
        for k in self.touch[a]:
            i, j = int(self.oc[k]), int(self.op[k])
            if self.intra[k]:
                if self.cam_dev[i] != a:
                    continue
                rj = residual_jacobians(cams_hat[i], pts_hat[j], self.uv[k], o.eps)
                if rj is None:  # R-N3d
                    continue
                r, Jc, Jl = rj
                w = self._rho_prime(r @ r)
                sc, sp = cpos[i], ppos[j]
                H[sc:sc + 9, sc:sc + 9] += w * Jc.T @ Jc
                H[sc:sc + 9, sp:sp + 3] += w * Jc.T @ Jl
                H[sp:sp + 3, sc:sc + 9] += w * Jl.T @ Jc
                H[sp:sp + 3, sp:sp + 3] += w * Jl.T @ Jl
                g[sc:sc + 9] += w * Jc.T @ r
                g[sp:sp + 3] += w * Jl.T @ r
            elif self.pt_dev[j] == a:
                c = self.coef(k, cams_hat, pts_hat)
                if c is None:
                    continue
                _, w, lam, gq = c
                sp = ppos[j]
                # eq. Q: Q(l) = w |lam l - g|^2 + a/2: gradient 2 w lam (lam l - g), Hessian 2 w lam^2 I
                H[sp:sp + 3, sp:sp + 3] += 2.0 * w * lam * lam * np.eye(3)
                g[sp:sp + 3] += 2.0 * w * lam * (lam * pts_hat[j] - gq)
        return H, g, ci, pj, cpos, ppos

    @staticmethod
    def lm_direction(H, g, mu):
        """The LM trial direction of reading R-N3c: (H + mu diag H) delta = -g solved by Jacobi-scaled Cholesky;
        None on a non-positive pivot (a failed trial)."""
        sc = 1.0 / np.sqrt(np.diag(H))
        Hs = H * np.outer(sc, sc)
        A = Hs + mu * np.diag(np.diag(Hs))
        try:
            L = np.linalg.cholesky(A)
        except np.linalg.LinAlgError:
            return None
        return np.linalg.solve(L.T, np.linalg.solve(L, -g * sc)) * sc

    def device_step(self, a, cams_hat, pts_hat):
        """argmin_{x^a} E^a(x^a | x_hat) approximated by one successful LM step from x_hat^a (R-N3a, R-N3c).
        Returns (cams, pts) with only device a's variables changed, and the accepted trial (-1: none)."""
        o = self.opt
        H, g, ci, pj, cpos, ppos = self.device_system(a, cams_hat, pts_hat)
        E0 = self.surrogate(cams_hat, pts_hat, cams_hat, pts_hat, [a])
        mu = o.lm_mu0
        for tau in range(o.lm_max_trials):
            delta = self.lm_direction(H, g, mu)
            if delta is None:
                mu *= o.lm_mu_up
                continue
            cams, pts = cams_hat.copy(), pts_hat.copy()
            for i in ci:
                s = cpos[int(i)]
                cams[i] = retract_camera(cams_hat[i], delta[s:s + 9])
            for j in pj:
                s = ppos[int(j)]
                pts[j] = pts_hat[j] + delta[s:s + 3]
            if self.surrogate(cams, pts, cams_hat, pts_hat, [a]) - E0 < 0:
                return cams, pts, tau
            mu *= o.lm_mu_up
        return cams_hat.copy(), pts_hat.copy(), -1

    def _rho_prime(self, s):
        return loss(self.opt.kind, self.opt.scale, s)[1]

    def solve_all(self, cams_hat, pts_hat):
        """x^{k+1} = argmin E(x | x_hat) device by device (eq. Esum: the device subproblems are independent)."""
        cams, pts = cams_hat.copy(), pts_hat.copy()
        trials = {}
        for a in self.devices:
            c, p, tr = self.device_step(a, cams_hat, pts_hat)
            cm, pm = self.cam_dev == a, self.pt_dev == a
            cams[cm], pts[pm] = c[cm], p[pm]
            trials[a] = tr
        return cams, pts, trials


def extrapolate(cams, cams_prev, pts, pts_prev, gamma):
    """x-bar^k (eqs. nesterov_x): R through ProjRot3D (eq. proj_rot3d), t, d, l linearly."""
    cb = cams + gamma * (cams - cams_prev)
    for i in range(cb.shape[0]):
        cb[i, :9] = proj_rot3d(cb[i, :9].reshape(3, 3)).reshape(9)
    return cb, pts + gamma * (pts - pts_prev)


def run(prob: Problem, iters: int):
    """Algorithm 1 with the coarse surrogate and the global restart test (reading D2).
    Returns (trace rows [F(x^k), F-bar^k, E_acc, restart, E_mm], final cams, final pts)."""
    o = prob.opt
    cams, pts = prob.cams0.copy(), prob.pts0.copy()
    cams_prev, pts_prev = cams.copy(), pts.copy()  # x^{-1} = x^0 (eq. Fainit)
    s = 1.0
    Fbar = prob.objective(cams, pts)  # F-bar^{-1} = F(x^0) (A18, global form)
    rows = []
    for _ in range(iters):
        s_next, gamma = schedule(s)  # eq. nesterov_scalar, Alg. 1
        if not o.accelerate:
            gamma = 0.0
        cb, lb = extrapolate(cams, cams_prev, pts, pts_prev, gamma)
        Fk = prob.objective(cams, pts)
        Fbar = (1.0 - o.eta) * Fbar + o.eta * Fk  # eq. lFak
        c_acc, l_acc, _ = prob.solve_all(cb, lb)  # eq. update_amm
        c_mm, l_mm, _ = prob.solve_all(cams, pts)  # eq. update_mm
        E_acc = prob.surrogate(c_acc, l_acc, cams, pts)  # eq. Eak, global form
        E_mm = prob.surrogate(c_mm, l_mm, cams, pts)
        restart = (E_acc > Fbar) if o.accelerate else True  # Alg. 1, strict ">"
        cams_prev, pts_prev = cams, pts
        cams, pts = (c_mm, l_mm) if restart else (c_acc, l_acc)
        rows.append([Fk, Fbar, E_acc, float(restart and o.accelerate), E_mm])
        s = s_next
    return np.array(rows), cams, pts


def normal_blocks(prob: Problem, cams, pts):
    """The Gauss-Newton blocks of sum_k F_k over ALL pairs (one device: every pair intra-device) at (cams, pts),
    reading R-N3a: per camera U_i = sum w J_c^T J_c, gc_i = sum w J_c^T r, F_cam_i = sum rho / 2; per point
    V_j = sum w J_l^T J_l, gl_j = sum w J_l^T r; per observation W_k = w J_c^T J_l.  Degenerate pairs add nothing
    (R-N3d).  The same terms device_step() adds for E' pairs."""
    o = prob.opt
    U, gc, Fc = np.zeros((prob.M, 9, 9)), np.zeros((prob.M, 9)), np.zeros(prob.M)
    V, gl, W = np.zeros((prob.N, 3, 3)), np.zeros((prob.N, 3)), np.zeros((prob.K, 9, 3))
    for k in range(prob.K):
        i, j = prob.oc[k], prob.op[k]
        rj = residual_jacobians(cams[i], pts[j], prob.uv[k], o.eps)
        if rj is None:
            continue
        r, Jc, Jl = rj
        rho, w = loss(o.kind, o.scale, r @ r)
        U[i] += w * Jc.T @ Jc
        gc[i] += w * Jc.T @ r
        Fc[i] += 0.5 * rho
        V[j] += w * Jl.T @ Jl
        gl[j] += w * Jl.T @ r
        W[k] = w * Jc.T @ Jl
    return U, gc, V, gl, W, Fc
