"""Pins for the oracle's surrogate (Prop. 1, eqs. P/Q/a/w/gamma/g) and its subproblem solvers (D3).

Fixed by: Proposition 1's equality/majorization, finite differences
(central, per-coordinate steps), the paper's gradient-equality at the anchor
(eq. gradFij), dense library least squares / linear solves, and a
Nelder-Mead minimiser of the camera surrogate.
"""
import numpy as np
import pytest
from scipy.optimize import minimize
from scipy.spatial.transform import Rotation

import oracle

rng = np.random.default_rng(99)
LOSSES = [oracle.LOSS_TRIVIAL, oracle.LOSS_HUBER, oracle.LOSS_CAUCHY]


def rand_rot(scale=None):
    return Rotation.random(random_state=rng.integers(1 << 31)).as_matrix()


def scene(n_obs=12, noise=3.0):
    """A camera looking down +z at points 5-20 units away, pixels from the model plus noise."""
    R = rand_rot()
    t = rng.normal(size=3)
    f = rng.uniform(600, 1200)
    k1, k2 = rng.uniform(-1, 1) * 0.1 / 1e6, rng.uniform(-1, 1) * 0.01 / 1e12
    cam = np.concatenate([R.ravel(), t, [f, f * k1, f * k2]])
    ls, us = [], []
    for _ in range(n_obs):
        u = rng.uniform([-700, -500], [700, 500])
        s = u @ u
        ray = np.array([u[0], u[1], f * (1 + k1 * s + k2 * s * s)])
        depth = rng.uniform(5, 20)
        ls.append(t + R @ (ray / ray[2] * depth))
        us.append(u + rng.normal(size=2) * noise)
    return cam, np.array(ls), np.array(us)


def perturb_cam(cam, ang=1e-3, dt=1e-2, dd=(1.0, 1e-5, 1e-11)):
    R = Rotation.from_rotvec(rng.normal(size=3) * ang).as_matrix() @ cam[:9].reshape(3, 3)
    return np.concatenate([R.ravel(), cam[9:12] + rng.normal(size=3) * dt, cam[12:] + rng.normal(size=3) * dd])


def retract(cam, delta):
    R = oracle.expmap(delta[:3]) @ cam[:9].reshape(3, 3)
    return np.concatenate([R.ravel(), cam[9:12] + delta[3:6], cam[12:] + delta[6:9]])


@pytest.mark.parametrize("kind", LOSSES)
def test_prop1_equality_and_majorization(kind):
    for _ in range(40):
        cam, ls, us = scene(n_obs=1, noise=rng.choice([0.5, 5.0, 40.0]))
        l, u = ls[0], us[0]
        coef = oracle.coefficients(cam, l, u, kind, 1.0)
        F = oracle.penalty(cam, l, u, kind, 1.0)
        # equality at the anchor, up to the cancellation of the g-form (Q21)
        assert oracle.P(coef, cam, u) + oracle.Q(coef, l) == pytest.approx(F, rel=1e-8, abs=1e-8)
        # majorization under perturbations (eq. majorize)
        for _ in range(50):
            c2 = perturb_cam(cam, ang=rng.choice([1e-4, 1e-2, 0.3]), dt=rng.choice([1e-3, 0.3]),
                             dd=(rng.choice([1.0, 50.0]), 1e-5, 1e-11))
            l2 = l + rng.normal(size=3) * rng.choice([1e-3, 0.5, 3.0])
            F2 = oracle.penalty(c2, l2, u, kind, 1.0)
            bound = oracle.P(coef, c2, u) + oracle.Q(coef, l2)
            assert F2 <= bound + 1e-8 * max(1.0, F2)


def test_coefficients_special_cases():
    cam, ls, us = scene(n_obs=5)
    for l, u in zip(ls, us):
        a, w, lam, g = oracle.coefficients(cam, l, u, oracle.LOSS_TRIVIAL, 1.0)
        assert a == 0.0 and w == 1.0  # trivial loss makes eq. a vanish
    # perfect observation: e = 0 -> a = 0, w = rho'(0) = 1 for every loss
    R, t, d = cam[:9].reshape(3, 3), cam[9:12], cam[12:]
    u = np.array([100.0, -50.0])
    p = oracle.ray(d, u)
    l = t + R @ p * 0.01
    for kind in LOSSES:
        a, w, lam, g = oracle.coefficients(cam, l, u, kind, 1.0)
        assert abs(a) < 1e-12 and w == pytest.approx(1.0, abs=1e-12)
        assert lam == pytest.approx(100.0, rel=1e-12)  # l - t = R p / 100


def tangent_steps(cam):
    d = cam[12:]
    return np.array([1e-6] * 3 + [1e-6] * 3 + [1e-6 * max(1, abs(d[0])), 1e-12, 1e-18])


@pytest.mark.parametrize("kind", LOSSES)
def test_camera_gradient_matches_fd_of_objective(kind):
    # eq. gradFij: at the anchor the surrogate's gradient equals that of F.  The oracle's g
    # (from its analytic Jacobian) is compared with central differences of sum_j F_ij on the tangent.
    opt = oracle.options(loss=kind, scale=1.0)
    for _ in range(10):
        cam, ls, us = scene(n_obs=15, noise=2.0)
        H, g = oracle.camera_normal_equations(cam, ls, us, opt)
        steps = tangent_steps(cam)
        fd = np.zeros(9)
        for k in range(9):
            dp = np.zeros(9)
            dp[k] = steps[k]
            Fp = sum(oracle.penalty(retract(cam, dp), l, u, kind, 1.0) for l, u in zip(ls, us))
            Fm = sum(oracle.penalty(retract(cam, -dp), l, u, kind, 1.0) for l, u in zip(ls, us))
            fd[k] = (Fp - Fm) / (2 * steps[k])
        scale = np.abs(g) + np.abs(fd) + 1e-6 * np.linalg.norm(g * steps) / steps
        assert np.all(np.abs(g - fd) <= 2e-5 * scale + 1e-8), (g, fd)


@pytest.mark.parametrize("kind", LOSSES)
def test_camera_hessian_is_gauss_newton_of_fd_jacobian(kind):
    opt = oracle.options(loss=kind, scale=1.0, xi=1e-4)
    cam, ls, us = scene(n_obs=10, noise=2.0)
    H, g = oracle.camera_normal_equations(cam, ls, us, opt)
    steps = tangent_steps(cam)
    Ht = np.diag([2 * opt.xi] * 3 + [opt.xi] * 6)
    for l, u in zip(ls, us):
        a, w, lam, gg = oracle.coefficients(cam, l, u, kind, 1.0)

        def r(c):  # the vector inside eq. P: R p(d) + lambda t - g
            return c[:9].reshape(3, 3) @ oracle.ray(c[12:], u) + lam * c[9:12] - gg
        J = np.zeros((3, 9))
        for k in range(9):
            dp = np.zeros(9)
            dp[k] = steps[k]
            J[:, k] = (r(retract(cam, dp)) - r(retract(cam, -dp))) / (2 * steps[k])
        Ht += 2 * w * J.T @ J
    D = np.sqrt(np.diag(Ht))
    np.testing.assert_allclose(H / np.outer(D, D), Ht / np.outer(D, D), atol=1e-6)


@pytest.mark.parametrize("kind", LOSSES)
def test_camera_lm_step_vs_dense_least_squares(kind):
    # The accepted trial is the Marquardt step (H + mu diag H) delta = -g; rebuild it with numpy's dense
    # least squares on the stacked sqrt(2w) J system (independent textbook routine), and check the decrease
    # against the literal surrogate sum_j P_j + xi/2 ||c - c_hat||^2 (eq. P, eq. Ealpha).
    opt = oracle.options(loss=kind, scale=1.0)
    for _ in range(8):
        cam, ls, us = scene(n_obs=20, noise=2.0)
        anchor = perturb_cam(cam, ang=2e-3, dt=5e-3, dd=(2.0, 0, 0))
        out, trial, dP = oracle.camera_solve(anchor, ls, us, opt)
        assert trial >= 0 and dP < 0
        H, g = oracle.camera_normal_equations(anchor, ls, us, opt)
        mu = opt.lm_mu0 * opt.lm_mu_up ** trial
        # stacked system: [sqrt(H) ; sqrt(mu diag H)] delta = [-(sqrt H)^-T g ; 0]
        Lh = np.linalg.cholesky(H)
        A = np.vstack([Lh.T, np.diag(np.sqrt(mu * np.diag(H)))])
        b = np.concatenate([-np.linalg.solve(Lh, g), np.zeros(9)])
        delta, *_ = np.linalg.lstsq(A, b, rcond=None)
        dtheta = Rotation.from_matrix(out[:9].reshape(3, 3) @ anchor[:9].reshape(3, 3).T).as_rotvec()
        got = np.concatenate([dtheta, out[9:12] - anchor[9:12], out[12:] - anchor[12:]])
        np.testing.assert_allclose(got, delta, rtol=1e-6, atol=1e-9 * np.abs(delta).max())
        # literal decrease, g-form P (with its cancellation) vs the anchor-relative dP
        lit = 0.0
        for l, u in zip(ls, us):
            coef = oracle.coefficients(anchor, l, u, kind, 1.0)
            lit += oracle.P(coef, out, u) - oracle.P(coef, anchor, u)
        lit += 0.5 * opt.xi * np.sum((out - anchor) ** 2)
        assert dP == pytest.approx(lit, rel=1e-6, abs=1e-6)


def test_camera_lm_moves_toward_nelder_mead_minimiser():
    # Brute force on a tiny subproblem: the exact minimiser of the camera surrogate by Nelder-Mead;
    # one LM step must decrease it and move the camera closer to the minimiser.
    opt = oracle.options(loss=oracle.LOSS_TRIVIAL)
    cam, ls, us = scene(n_obs=3, noise=0.5)
    anchor = perturb_cam(cam, ang=1e-3, dt=1e-3, dd=(0.5, 0, 0))
    coefs = [oracle.coefficients(anchor, l, u) for l, u in zip(ls, us)]
    sc = np.array([1e-3] * 3 + [1e-3] * 3 + [1.0, 1e-6, 1e-12])

    def E(z):
        c = retract(anchor, z * sc)
        return sum(oracle.P(cf, c, u) for cf, u in zip(coefs, us)) + 0.5 * opt.xi * np.sum((c - anchor) ** 2)
    res = minimize(E, np.zeros(9), method="Nelder-Mead", options=dict(xatol=1e-10, fatol=1e-14, maxiter=40000,
                                                                       maxfev=40000))
    out, trial, dP = oracle.camera_solve(anchor, ls, us, opt)
    z_lm = np.concatenate([Rotation.from_matrix(out[:9].reshape(3, 3) @ anchor[:9].reshape(3, 3).T).as_rotvec(),
                           out[9:12] - anchor[9:12], out[12:] - anchor[12:]]) / sc
    assert E(z_lm) < E(np.zeros(9))
    assert np.linalg.norm(z_lm - res.x) < np.linalg.norm(res.x)


@pytest.mark.parametrize("kind", LOSSES)
def test_point_solve_closed_form(kind):
    # Exact minimiser of sum_i Q_ij(l) + xi/2 ||l - l_hat||^2 (eq. Q, eq. Ealpha): dense 3x3 solve of the
    # normal equations built from eq. Q's quadratic form, and a zero finite-difference gradient.
    opt = oracle.options(loss=kind, scale=1.0)
    for _ in range(20):
        l_hat = rng.normal(size=3) * 3 + np.array([0, 0, 10.0])
        n = rng.integers(1, 9)
        cams = []
        us = []
        for _ in range(n):
            R = Rotation.from_rotvec(rng.normal(size=3) * 0.2).as_matrix()
            t = rng.normal(size=3)
            f = rng.uniform(600, 1200)
            cams.append(np.concatenate([R.ravel(), t, [f, 1e-5 * rng.normal(), 1e-12 * rng.normal()]]))
            us.append(rng.uniform(-300, 300, size=2))
        cams = np.array(cams)
        us = np.array(us)
        out = oracle.point_solve(l_hat, cams, us, opt)
        A = opt.xi * np.eye(3)
        b = opt.xi * l_hat
        coefs = [oracle.coefficients(c, l_hat, u, kind, 1.0) for c, u in zip(cams, us)]
        for a, w, lam, g in coefs:
            A += 2 * w * lam * lam * np.eye(3)
            b += 2 * w * lam * g
        np.testing.assert_allclose(out, np.linalg.solve(A, b), rtol=1e-10, atol=1e-10)

        def obj(l):
            return sum(oracle.Q(cf, l) for cf in coefs) + 0.5 * opt.xi * np.sum((l - l_hat) ** 2)
        h = 1e-5
        grad = np.array([(obj(out + h * e) - obj(out - h * e)) / (2 * h) for e in np.eye(3)])
        scale = max(1.0, np.abs([(obj(l_hat + h * e) - obj(l_hat - h * e)) / (2 * h) for e in np.eye(3)]).max())
        assert np.abs(grad).max() <= 1e-5 * scale
