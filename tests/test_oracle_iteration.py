"""Pins for the oracle's acceleration (§5) and the full iteration (Algorithm 1).

Fixed by: closed-form schedule constants (eq. nesterov_scalar), Horn's quaternion
method for ProjRot3D (an independent textbook routine), the convergence theory of
App. C.3.1 (F-bar nonincreasing, the descent inequality eq. FklFk0),
MM monotonicity, the k=0 special case, the noiseless fixed point,
Prop. 3 (gradient -> 0), and a literal evaluation of eq. Eak with eqs. P/Q.
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import gen
import oracle

rng = np.random.default_rng(7)
PHI = (1 + math.sqrt(5)) / 2
# App. A of SURVEY.md: gamma_k for k = 0..5, s_1, s_2 (closed-form evaluation of eq. nesterov_scalar)
GAMMAS = [0.0, 0.281753525125, 0.434042782780, 0.531063805404, 0.598778594056, 0.648923326122]


def test_schedule_constants():
    s = 1.0
    for k, gexp in enumerate(GAMMAS):
        s_next, g = oracle.schedule(s)
        assert g == pytest.approx(gexp, abs=5e-13)
        if k == 0:
            assert s_next == pytest.approx(PHI, abs=1e-15)
        if k == 1:
            assert s_next == pytest.approx(2.193527085331, abs=1e-12)
        s = s_next
    # gamma in [0,1) for any s >= 1 (eq. gamma_bnd); s grows like k/2
    s = 1.0
    for k in range(1000):
        s_next, g = oracle.schedule(s)
        assert 0.0 <= g < 1.0 and s_next > s
        s = s_next
    assert 490 < s < 510


def horn_projection(M):
    """ProjRot3D by Horn's closed form: the unit quaternion maximising tr(R^T M) is the top eigenvector
    of the 4x4 symmetric matrix built from M (Horn 1987)."""
    Sxx, Sxy, Sxz, Syx, Syy, Syz, Szx, Szy, Szz = M.T.ravel()
    N = np.array([[Sxx + Syy + Szz, Syz - Szy, Szx - Sxz, Sxy - Syx],
                  [Syz - Szy, Sxx - Syy - Szz, Sxy + Syx, Szx + Sxz],
                  [Szx - Sxz, Sxy + Syx, -Sxx + Syy - Szz, Syz + Szy],
                  [Sxy - Syx, Szx + Sxz, Syz + Szy, -Sxx - Syy + Szz]])
    w, V = np.linalg.eigh(N)
    q = V[:, -1]
    return Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()


def test_proj_rot3d():
    for _ in range(200):
        R = Rotation.random(random_state=rng.integers(1 << 31)).as_matrix()
        np.testing.assert_allclose(oracle.proj_rot3d(R), R, atol=1e-14)          # ProjRot3D(R) = R
        np.testing.assert_allclose(oracle.proj_rot3d(2.0 * R), R, atol=1e-14)    # ProjRot3D(2R) = R
        M = R + rng.normal(size=(3, 3)) * rng.choice([1e-6, 0.1, 1.0])
        P = oracle.proj_rot3d(M)
        np.testing.assert_allclose(P @ P.T, np.eye(3), atol=1e-13)
        assert np.linalg.det(P) == pytest.approx(1.0, abs=1e-13)
        H = horn_projection(M)
        if np.linalg.norm(P - H) > 1e-9:  # only a genuine tie may disagree
            assert np.sum((P - M) ** 2) == pytest.approx(np.sum((H - M) ** 2), rel=1e-12)
        # sampled argmin: no random rotation is closer
        for _ in range(20):
            Q = Rotation.random(random_state=rng.integers(1 << 31)).as_matrix()
            assert np.sum((P - M) ** 2) <= np.sum((Q - M) ** 2) + 1e-12
    # det(M) < 0: the flip lands on the smallest singular direction
    M = np.diag([3.0, 2.0, -1.0])
    np.testing.assert_allclose(oracle.proj_rot3d(M), np.eye(3), atol=1e-14)


def run(name, n, **kw):
    p = gen.generate(name)
    o = oracle.Oracle(p, **kw)
    return p, o, o.iterate(n)


@pytest.mark.parametrize("name", ["tiny_seq", "small_huber", "small_cauchy"])
@pytest.mark.parametrize("eta", [0.1, 1.0])
def test_iteration_invariants(name, eta):
    xi = 1e-4
    p, o, tr = run(name, 30, eta=eta)
    F, Fb, Eacc, rs, Emm, st = (tr[:, c] for c in (oracle.TR_F, oracle.TR_FBAR, oracle.TR_EACC, oracle.TR_RESTART,
                                                    oracle.TR_EMM, oracle.TR_STEP2))
    tol = 1e-12 * F[0]
    assert tr[0, oracle.TR_GAMMA] == 0.0 and rs[0] == 0          # k = 0: gamma_0 = 0, no restart
    assert np.all(np.diff(Fb) <= tol)                           # F-bar nonincreasing (App. C.3.1)
    assert np.all(F[1:] + 0.5 * xi * st[:-1] <= Fb[:-1] + tol)  # eq. FklFk0
    assert np.all(Emm <= F + tol)                                # MM step never increases the surrogate
    assert np.all((Eacc > Fb) == (rs == 1))                      # restart test (Alg. 1), strict ">"
    if eta == 1.0:
        assert np.all(np.diff(F) <= tol)                         # F-bar = F: literal monotonicity
        assert rs.sum() > 0                                      # restarts are exercised
    assert F[-1] < F[0]


def test_unaccelerated_mm_is_monotone():
    # DUBA: gamma = 0, always the MM update -> F(x^{k+1}) <= F(x^k)
    p, o, tr = run("small_huber", 20, accelerate=0)
    F = tr[:, oracle.TR_F]
    assert np.all(np.diff(F) <= 1e-12 * F[0])
    assert np.all(tr[:, oracle.TR_GAMMA] == 0)


def literal_E(o, p, xk_c, xk_l, x_c, x_l, kind, xi):
    """eq. Ealpha (all pairs majorized, D1): sum_E [P_ij(c_i|x^k) + Q_ij(l_j|x^k)] + xi/2 ||x - x^k||^2."""
    tot = 0.0
    for k in range(p.K):
        i, j = p.obs_cam[k], p.obs_pt[k]
        coef = oracle.coefficients(xk_c[i], xk_l[j], p.obs_uv[k], kind, p.loss_scale)
        tot += oracle.P(coef, x_c[i], p.obs_uv[k]) + oracle.Q(coef, x_l[j])
    return tot + 0.5 * xi * (np.sum((x_c - xk_c) ** 2) + np.sum((x_l - xk_l) ** 2))


def test_E_acc_matches_literal_surrogate():
    # eq. Eak (global form): E_acc = E(x^{k+1} | x^k) when no restart fires; evaluated literally with eqs. P/Q
    p = gen.generate("tiny_seq")
    o = oracle.Oracle(p)
    c0, l0 = o.state(0)
    tr = o.iterate(3)
    assert tr[:, oracle.TR_RESTART].sum() == 0
    o2 = oracle.Oracle(p)
    for k in range(3):
        ck, lk = o2.state(0)
        o2.iterate(1)
        c1, l1 = o2.state(0)
        E = literal_E(o2, p, ck, lk, c1, l1, p.loss, 1e-4)
        assert tr[k, oracle.TR_EACC] == pytest.approx(E, rel=1e-9)
        if k < 2:  # F(x^{k+1}) + xi/2 ||x^{k+1} - x^k||^2 <= E(x^{k+1}|x^k) (Prop. 2 with the proximal term)
            assert tr[k + 1, oracle.TR_F] + 0.5 * 1e-4 * tr[k, oracle.TR_STEP2] <= E * (1 + 1e-12)


def test_noiseless_ground_truth_is_fixed_point():
    p = gen.generate("small_huber", noise_px=0.0, outlier_frac=0.0, init_scale=0.0)
    o = oracle.Oracle(p)
    tr = o.iterate(5)
    assert np.all(tr[:, oracle.TR_F] < 1e-12 * p.K)
    c, l = o.state(0)
    np.testing.assert_allclose(l, p.gt_pts, atol=1e-8)
    np.testing.assert_allclose(oracle.native_to_bal(c), p.gt_cams, rtol=1e-8, atol=1e-8)


def riemannian_grad_norm(p, cams, pts, kind):
    """||grad F|| by central differences on the tangent: rotations by left Exp, others additive."""
    def F(c, l):
        tot = 0.0
        for k in range(p.K):
            tot += oracle.penalty(c[p.obs_cam[k]], l[p.obs_pt[k]], p.obs_uv[k], kind, p.loss_scale)
        return tot
    g2 = 0.0
    for i in range(p.M):
        sc = [1e-6] * 6 + [1e-6 * cams[i, 12], 1e-12, 1e-18]
        natural = [1.0] * 7 + [1e-6, 1e-12]  # gradients in d2, d3 scaled by |u|^-2, |u|^-4 (|u|^2 ~ 1e6)
        for k in range(9):
            cp, cm = cams.copy(), cams.copy()
            for c, sgn in ((cp, 1), (cm, -1)):
                d = np.zeros(9)
                d[k] = sgn * sc[k]
                R = oracle.expmap(d[:3]) @ cams[i, :9].reshape(3, 3)
                c[i] = np.concatenate([R.ravel(), cams[i, 9:12] + d[3:6], cams[i, 12:] + d[6:]])
            g = (F(cp, pts) - F(cm, pts)) / (2 * sc[k])
            g2 += (g * natural[k]) ** 2
    for j in range(p.N):
        for k in range(3):
            lp, lm = pts.copy(), pts.copy()
            lp[j, k] += 1e-6
            lm[j, k] -= 1e-6
            g2 += ((F(cams, lp) - F(cams, lm)) / 2e-6) ** 2
    return math.sqrt(g2)


@pytest.mark.slow
def test_convergence_to_critical_point():
    # Prop. 3: on a noiseless problem F -> 0 and the Riemannian gradient norm -> 0
    p = gen.generate("tiny_seq", noise_px=0.0, outlier_frac=0.0)
    o = oracle.Oracle(p)
    c0, l0 = o.state(0)
    g0 = riemannian_grad_norm(p, c0, l0, p.loss)
    tr = o.iterate(1500)
    F = tr[:, oracle.TR_F]
    c, l = o.state(0)
    g1 = riemannian_grad_norm(p, c, l, p.loss)
    assert F[-1] < 1e-5 * F[0]
    assert g1 < 1e-4 * g0
    assert np.all(np.diff(tr[:, oracle.TR_FBAR]) <= 1e-12 * F[0])
