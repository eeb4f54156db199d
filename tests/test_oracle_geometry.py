"""Pins for the oracle's geometry and loss (§3, Assumption 1).

Each check is fixed by something other than the oracle itself: worked values that
follow by hand from the paper's equations (tests/golden/worked_values.json),
closed forms, library routines (scipy minimisation / rotations), invariants.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.optimize import minimize_scalar
from scipy.spatial.transform import Rotation

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))
rng = np.random.default_rng(1234)


def rand_rot():
    return Rotation.random(random_state=rng.integers(1 << 31)).as_matrix()


def rand_cam():
    R = rand_rot()
    t = rng.normal(size=3) * 3
    d = np.array([rng.uniform(500, 1500), rng.uniform(-1, 1) * 1e-4 * 1000, rng.uniform(-1, 1) * 1e-14 * 1000])
    return np.concatenate([R.ravel(), t, d])


def test_ray_worked_values():
    for case in GOLD["ray"]:
        np.testing.assert_array_equal(oracle.ray(case["d"], case["u"]), case["p"])


def test_ray_random_horner():
    for _ in range(200):
        d = rng.normal(size=3)
        u = rng.normal(size=2) * 100
        s = u @ u
        p = oracle.ray(d, u)
        assert p[0] == u[0] and p[1] == u[1]
        assert abs(p[2] - (d[0] + s * (d[1] + s * d[2]))) <= 1e-12 * (abs(d[0]) + abs(d[1]) * s + abs(d[2]) * s * s)


def test_optimal_scale_worked_values():
    for case in GOLD["optimal_scale"]:
        lam = oracle.optimal_scale(np.array(case["R"]), case["t"], case["l"], case["p"])
        assert lam == pytest.approx(case["lambda"], abs=1e-15)


def test_optimal_scale_is_argmin_brent():
    # eq. error_opt: lambda minimises ||p - lambda R^T (l - t)||^2 — checked by a 1-D library minimiser
    for _ in range(100):
        R, t, l = rand_rot(), rng.normal(size=3), rng.normal(size=3) * 5
        p = rng.normal(size=3)
        lam = oracle.optimal_scale(R, t, l, p)
        f = lambda x: float(np.sum((p - x * R.T @ (l - t)) ** 2))
        res = minimize_scalar(f, bracket=(-10, 10), tol=1e-14)
        assert lam == pytest.approx(res.x, rel=1e-6, abs=1e-8)


def test_degenerate_pair_rejected():
    # Assumption 2: ||l - t|| > eps required
    R, t = np.eye(3), np.zeros(3)
    assert oracle.optimal_scale(R, t, np.array([0, 0, 1e-9]), np.ones(3)) is None
    assert oracle.reprojection_error(R, t, np.zeros(3), np.ones(3)) is None


def test_reprojection_error_special_cases():
    R, t, l = np.eye(3), np.zeros(3), np.array([0.0, 0.0, 1.0])
    np.testing.assert_allclose(oracle.reprojection_error(R, t, l, [0, 0, 3.0]), 0, atol=1e-15)  # parallel -> 0
    np.testing.assert_allclose(oracle.reprojection_error(R, t, l, [2.0, -1.0, 0]), [2, -1, 0], atol=1e-15)  # orth -> p


def test_reprojection_error_invariants():
    for _ in range(300):
        R, t, l = rand_rot(), rng.normal(size=3), rng.normal(size=3) * 4
        p = rng.normal(size=3) * 10
        e = oracle.reprojection_error(R, t, l, p)
        v = R.T @ (l - t)
        assert abs(e @ v) <= 1e-12 * np.linalg.norm(p) * np.linalg.norm(v)       # normal plane (Fig. 2)
        assert np.linalg.norm(e) <= np.linalg.norm(p) * (1 + 1e-15)              # projection shrinks
        # ||e||^2 is the minimum over lambda: brute-force check of 20 random lambdas
        for lam in rng.normal(size=20) * 5:
            assert e @ e <= np.sum((p - lam * v) ** 2) * (1 + 1e-14) + 1e-14


def test_reprojection_error_gauge_invariance():
    # ||e|| is invariant under a global rigid motion (R, t, l) -> (Q R, Q t + c, Q l + c)
    for _ in range(50):
        R, t, l, p = rand_rot(), rng.normal(size=3), rng.normal(size=3) * 4, rng.normal(size=3)
        Qr, c = rand_rot(), rng.normal(size=3) * 10
        e1 = oracle.reprojection_error(R, t, l, p)
        e2 = oracle.reprojection_error(Qr @ R, Qr @ t + c, Qr @ l + c, p)
        assert np.linalg.norm(e1) == pytest.approx(np.linalg.norm(e2), rel=1e-10, abs=1e-12)


@pytest.mark.parametrize("kind", [oracle.LOSS_TRIVIAL, oracle.LOSS_HUBER, oracle.LOSS_CAUCHY])
def test_loss_assumption1(kind):
    # Assumption 1: rho(0) = 0, rho'(0) = 1, 0 <= rho' <= 1, concave, nondecreasing, rho' = d rho / ds
    for scale in (0.5, 1.0, 2.0):
        r0, d0 = oracle.loss(kind, scale, 0.0)
        assert r0 == 0.0 and d0 == 1.0
        grid = np.concatenate([np.linspace(0, 10, 401), np.geomspace(10, 1e6, 100)])
        vals = np.array([oracle.loss(kind, scale, s) for s in grid])
        assert np.all(vals[:, 1] >= 0) and np.all(vals[:, 1] <= 1)
        assert np.all(np.diff(vals[:, 0]) >= -1e-12)
        for a, b in zip(grid[:-1], grid[1:]):  # midpoint concavity
            m = oracle.loss(kind, scale, 0.5 * (a + b))[0]
            assert m >= 0.5 * (oracle.loss(kind, scale, a)[0] + oracle.loss(kind, scale, b)[0]) - 1e-9 * (1 + m)
        for s in rng.uniform(0.01, 50, 50):  # derivative by central differences
            h = 1e-6 * max(1.0, s)
            fd = (oracle.loss(kind, scale, s + h)[0] - oracle.loss(kind, scale, s - h)[0]) / (2 * h)
            assert oracle.loss(kind, scale, s)[1] == pytest.approx(fd, rel=1e-6, abs=1e-9)


def test_loss_worked_values():
    for case in GOLD["loss"]:
        r, d = oracle.loss(case["kind"], case["scale"], case["s"])
        assert r == pytest.approx(case["rho"], rel=1e-14)
        assert d == pytest.approx(case["drho"], rel=1e-14)


def test_penalty_worked_values():
    for case in GOLD["penalty"]:
        F = oracle.penalty(np.array(case["cam"], float), case["l"], case["u"], case["kind"], case["scale"])
        assert F == pytest.approx(case["F"], rel=1e-14, abs=1e-15)


def test_expmap_and_bal_conversion_vs_scipy():
    for _ in range(100):
        w = rng.normal(size=3) * rng.choice([1e-10, 1e-3, 1.0, 3.0])
        np.testing.assert_allclose(oracle.expmap(w), Rotation.from_rotvec(w).as_matrix(), atol=1e-14)
    np.testing.assert_allclose(oracle.expmap([math.pi, 0, 0]), np.diag([1.0, -1.0, -1.0]), atol=1e-15)
    bal = np.concatenate([rng.normal(size=(20, 3)), rng.normal(size=(20, 3)) * 5,
                          np.column_stack([rng.uniform(500, 1500, 20), rng.normal(size=20) * 1e-7,
                                           rng.normal(size=20) * 1e-14])], axis=1)
    nat = oracle.bal_to_native(bal)
    for b, c in zip(bal, nat):
        Rw2c = Rotation.from_rotvec(b[:3]).as_matrix()
        np.testing.assert_allclose(c[:9].reshape(3, 3), Rw2c.T, atol=1e-14)
        np.testing.assert_allclose(c[9:12], -Rw2c.T @ b[3:6], rtol=1e-13, atol=1e-13)   # camera centre
        np.testing.assert_allclose(c[12:], [b[6], b[6] * b[7], b[6] * b[8]], rtol=1e-15)  # d = (f, f k1, f k2)
    back = oracle.native_to_bal(nat)
    np.testing.assert_allclose(Rotation.from_rotvec(back[:, :3]).as_matrix(),
                               Rotation.from_rotvec(bal[:, :3]).as_matrix(), atol=1e-13)
    np.testing.assert_allclose(back[:, 3:], bal[:, 3:], rtol=1e-12, atol=1e-12)
