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


# ---------------------------------------------------------------- extrapolation (eqs. nesterov_R/t/d/l)
import dataclasses
import json
import os

EXTRAP = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))["extrapolate"]


def rz(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


@pytest.mark.parametrize("case", range(len(EXTRAP)))
def test_camera_extrapolation_worked_value(case):
    # tests/golden/worked_values.json "extrapolate": R^k = Rz(theta) R0, R^{k-1} = R0 -> x-bar rotation Rz(phi) R0
    v = EXTRAP[case]
    R0 = Rotation.from_rotvec([0.3, -1.1, 0.7]).as_matrix()
    c, cp = np.zeros(15), np.zeros(15)
    c[:9], cp[:9] = (rz(v["theta"]) @ R0).ravel(), R0.ravel()
    c[9:12], cp[9:12] = v.get("t", [1.0, 2.0, 3.0]), v.get("t_prev", [1.0, 2.0, 3.0])
    c[12:], cp[12:] = v.get("d", [800.0, 0.0, 0.0]), v.get("d_prev", [800.0, 0.0, 0.0])
    out = oracle.extrapolate_camera(c, cp, v["gamma"])
    np.testing.assert_allclose(out[:9].reshape(3, 3), rz(v["phi"]) @ R0, atol=2e-15)
    if "t_bar" in v:
        np.testing.assert_allclose(out[9:12], v["t_bar"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(out[12:], v["d_bar"], rtol=1e-15)
        # eq. nesterov_l, the same linear rule for a point
        np.testing.assert_allclose(oracle.extrapolate_point(v["t"], v["t_prev"], v["gamma"]), v["t_bar"], atol=1e-15)


def with_isolated(p):
    """p plus one camera and one point that no observation touches (their subproblems are the proximal term
    alone, minimised at the anchor: the accelerated candidate of each is x-bar itself)."""
    cams = np.vstack([p.cams, p.cams[:1]])
    pts = np.vstack([p.pts, p.pts[:1] + 1.0])
    return dataclasses.replace(p, cams=cams, pts=pts)


def isolated_setup(p, Rk, Rkm1, s=PHI):
    """Oracle on p + isolated camera / point, x^k = x^0 except the isolated camera rotation Rk (x^{k-1}: Rkm1)
    and the isolated point moved by (0.5, -0.25, 2); s^{(k)} = s, F-bar^{(k-1)} large (no restart)."""
    q = with_isolated(p)
    o = oracle.Oracle(q)
    ck, lk = o.state(0)
    ckm1, lkm1 = ck.copy(), lk.copy()
    ck[-1, :9], ckm1[-1, :9] = np.ravel(Rk), np.ravel(Rkm1)
    ck[-1, 9:12], ckm1[-1, 9:12] = [1.0, 2.0, 3.0], [0.5, 2.5, 3.0]
    lkm1[-1] = lk[-1] - [0.5, -0.25, 2.0]
    o.set_state(0, ck, lk)
    o.set_state(1, ckm1, lkm1)
    o.set_schedule(s, 1e30)
    return o, ck, lk, ckm1, lkm1


def test_isolated_camera_moves_by_its_extrapolation():
    # Alg. 1 L407-414 on an isolated camera and point: no restart (F-bar huge), so x^{k+1} = x_acc = x-bar^k, and
    # x-bar^k is fixed in closed form by the worked value (gamma_1 from s = phi)
    v = EXTRAP[0]
    R0 = Rotation.from_rotvec([0.3, -1.1, 0.7]).as_matrix()
    o, ck, lk, ckm1, lkm1 = isolated_setup(gen.generate("tiny_seq"), rz(v["theta"]) @ R0, R0)
    tr = o.iterate(1)
    assert tr[0, oracle.TR_RESTART] == 0
    assert tr[0, oracle.TR_GAMMA] == pytest.approx(v["gamma"], abs=1e-12)
    c1, l1 = o.state(0)
    np.testing.assert_allclose(c1[-1, :9].reshape(3, 3), rz(v["phi"]) @ R0, atol=1e-14)
    np.testing.assert_allclose(c1[-1, 9:12], v["t_bar"], atol=1e-14)
    np.testing.assert_allclose(l1[-1], lk[-1] + v["gamma"] * np.array([0.5, -0.25, 2.0]), atol=1e-14)
    # the other variables are unaffected by the isolated pair of variables: same iterate as without them
    p = gen.generate("tiny_seq")
    ref = oracle.Oracle(p)
    ref.set_schedule(PHI, 1e30)
    ref.iterate(1)
    cr, lr = ref.state(0)
    np.testing.assert_array_equal(c1[:-1], cr)
    np.testing.assert_array_equal(l1[:-1], lr)


def test_isolated_camera_extrapolation_with_negative_determinant():
    # ProjRot3D's det < 0 case (eq. proj_rot3d, Q14) inside the iteration: R^k = R^{k-1} = U diag(3,2,-1/2) V^T
    # (not a rotation, so only reachable through set_state) -> x-bar rotation = U V^T in closed form (the sign
    # flip lands on the smallest singular direction)
    U = Rotation.from_rotvec([0.2, 0.5, -0.4]).as_matrix()
    V = Rotation.from_rotvec([-1.0, 0.3, 0.8]).as_matrix()
    M = U @ np.diag([3.0, 2.0, -0.5]) @ V.T
    assert np.linalg.det(M) < 0
    o, *_ = isolated_setup(gen.generate("tiny_seq"), M, M)
    tr = o.iterate(1)
    assert tr[0, oracle.TR_RESTART] == 0
    c1, _ = o.state(0)
    np.testing.assert_allclose(c1[-1, :9].reshape(3, 3), U @ V.T, atol=1e-13)


@pytest.mark.parametrize("loss", [oracle.LOSS_TRIVIAL, oracle.LOSS_HUBER])
def test_acceleration_reaches_F_delta_sooner(loss):
    # DABA reaches F_Delta (eq. Fdelta, Delta = 2.5e-4 as in the tables' captions) in fewer
    # iterations than its unaccelerated ablation DUBA; F_ref = the best F either reaches in 600 iterations
    p = gen.generate("tiny_seq", loss=loss, outlier_frac=0.03 if loss else 0.0)
    Fa = oracle.Oracle(p).iterate(600)[:, oracle.TR_F]
    Fd = oracle.Oracle(p, accelerate=0).iterate(600)[:, oracle.TR_F]
    Fref = min(Fa.min(), Fd.min())
    Fdelta = Fref + 2.5e-4 * (Fa[0] - Fref)
    ia = int(np.argmax(Fa <= Fdelta))
    assert Fa[ia] <= Fdelta
    idd = int(np.argmax(Fd <= Fdelta)) if (Fd <= Fdelta).any() else 10 ** 9
    assert 2 * ia < idd, (ia, idd)
