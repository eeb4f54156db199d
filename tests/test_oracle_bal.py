"""Pins for the BAL oracle (oracle/bal.py): parsing, BAL's forward model, the pixel metric
of Table 2 and the BAL <-> paper convention map (reading Q15).

Fixed by things other than the oracle itself:
  - hand-evaluated fixtures (tests/golden/bal_*.txt / .json, exact fractions);
  - BAL's pinhole special case (k1 = k2 = 0) equals the homogeneous projection K [R | t] X with K = diag(f, f, -1);
  - the converted problem satisfies the PAPER's model (the C++ oracle's eq. error / lambdaij, independent code):
    a noiseless distortion-free BAL scene has e_ij = 0 and lambda_ij > 0 for every observation, F(x) = 0;
  - the intrinsics map is a series reversion exact through O(|u|^4): the remaining ray mismatch shrinks like
    |u|^7 (a dropped or wrong k2' term leaves |u|^5);
  - bal_to_paper o paper_to_bal is the identity.
"""
import json
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import gen
import oracle
from oracle import bal as B

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bal_scene(M=6, N=60, seed=0, k1=0.0, k2=0.0, noise=0.0, f=800.0):
    """Cameras on a sphere of radius 6-9 looking at the origin (BAL: down -z), points in the unit ball, every
    camera sees every point; observations from BAL's forward model (oracle.bal.bal_project) + pixel noise."""
    r = np.random.default_rng(seed)
    cams = np.empty((M, 9))
    for i in range(M):
        c = r.normal(size=3)
        c *= r.uniform(6, 9) / np.linalg.norm(c)
        w = -c / np.linalg.norm(c)                      # viewing direction = camera -z
        x = np.cross(w, r.normal(size=3))
        x /= np.linalg.norm(x)
        y = np.cross(-w, x)
        Rw = np.stack([x, y, -w])                       # rows: camera axes in world coordinates
        cams[i, :3] = Rotation.from_matrix(Rw).as_rotvec()
        cams[i, 3:6] = -Rw @ c
        cams[i, 6:9] = f * r.uniform(0.9, 1.1), k1, k2
    pts = r.uniform(-1, 1, (N, 3)) * 0.6
    oc = np.repeat(np.arange(M, dtype=np.int32), N)
    op = np.tile(np.arange(N, dtype=np.int32), M)
    uv = np.concatenate([B.bal_project(cams[i], pts) for i in range(M)]) + r.normal(size=(M * N, 2)) * noise
    return cams, pts, oc, op, uv


def paper_F(cams_abi, pts, oc, op, uv):
    p = gen.Problem("bal", cams_abi, pts, oc, op, uv, cams_abi, pts, 0)
    return oracle.Oracle(p).objective()


def test_golden_minimal():
    # 1 camera at the origin, point (0,0,-1) in front of BAL's camera
    with open(os.path.join(GOLD, "bal_minimal.txt")) as f:
        cams, pts, oc, op, uv = B.parse_bal(f.read())
    assert (cams.shape, pts.shape, oc.tolist(), op.tolist()) == ((1, 9), (1, 3), [0], [0])
    assert B.mean_pixel_error(cams, pts, oc, op, uv) == (0.0, 0.0, 0, 1)
    c, u = B.bal_to_paper(cams, uv)
    nat = oracle.bal_to_native(c)[0]
    R, t, d = nat[:9].reshape(3, 3), nat[9:12], nat[12:15]
    p = oracle.ray(d, u[0])
    assert oracle.optimal_scale(R, t, pts[0], p) > 0
    np.testing.assert_allclose(oracle.reprojection_error(R, t, pts[0], p), 0, atol=1e-15)


def test_golden_two_views():
    with open(os.path.join(GOLD, "bal_two_views.json")) as f:
        g = json.load(f)
    with open(os.path.join(GOLD, "bal_two_views.txt")) as f:
        cams, pts, oc, op, uv = B.parse_bal(f.read())
    assert [len(cams), len(pts), len(oc)] == g["counts"]
    err, behind = B.pixel_residuals(cams, pts, oc, op, uv)
    np.testing.assert_allclose(err, g["abs_residuals"], rtol=0, atol=1e-12)
    s, s2, nb, n = B.mean_pixel_error(cams, pts, oc, op, uv)
    assert s / n == pytest.approx(g["mean"], abs=1e-12)
    assert s2 == pytest.approx(g["sum_sq"], abs=1e-11)
    assert nb == g["behind"]


@pytest.mark.parametrize("text,msg", [
    ("1 1 2\n0 0 0 0\n", "end of file"),
    ("1 1 1\n0 1 0 0\n" + "0 " * 9 + "0 0 -1\n", "out of range"),
    ("1 1 1\n0 0 0 0\n" + "0 " * 9 + "0 0 -1 7\n", "trailing"),
])
def test_parse_errors(text, msg):
    with pytest.raises(ValueError, match=msg):
        B.parse_bal(text)


def test_pinhole_is_the_homogeneous_projection():
    cams, pts, *_ = bal_scene(M=4, N=20, seed=3)
    for c in cams:
        Rw = Rotation.from_rotvec(c[:3]).as_matrix()
        Kmat = np.diag([c[6], c[6], -1.0])
        h = (Kmat @ np.hstack([Rw, c[3:6, None]]) @ np.vstack([pts.T, np.ones(len(pts))])).T
        np.testing.assert_allclose(B.bal_project(c, pts), h[:, :2] / h[:, 2:3], rtol=1e-13)


def test_radial_distortion_scales_along_the_ray():
    # u = f r(|p|) p: the same direction as the pinhole pixel, radius times 1 + k1 rho^2 + k2 rho^4
    cams, pts, *_ = bal_scene(M=3, N=30, seed=4)
    for c in cams:
        u0 = B.bal_project(c, pts)
        cd = c.copy()
        cd[7:9] = -0.3, 0.2
        ud = B.bal_project(cd, pts)
        rho = np.linalg.norm(u0, axis=1) / c[6]
        np.testing.assert_allclose(u0[:, 0] * ud[:, 1] - u0[:, 1] * ud[:, 0], 0, atol=1e-9)
        np.testing.assert_allclose(np.linalg.norm(ud, axis=1) / np.linalg.norm(u0, axis=1),
                                   1 - 0.3 * rho ** 2 + 0.2 * rho ** 4, rtol=1e-13)


def test_converted_scene_satisfies_the_paper_model():
    # noiseless, distortion-free BAL scene -> e_ij = 0 (eq. error) with lambda_ij > 0 (eq. lambdaij), F = 0
    cams, pts, oc, op, uv = bal_scene(seed=5)
    c, u = B.bal_to_paper(cams, uv)
    nat = oracle.bal_to_native(c)
    F0 = paper_F(c, pts, oc, op, u)
    assert F0 < 1e-18 * len(oc) * 800 ** 2
    for q in range(0, len(oc), 7):
        n = nat[oc[q]]
        R, t, d = n[:9].reshape(3, 3), n[9:12], n[12:15]
        p = oracle.ray(d, u[q])
        assert oracle.optimal_scale(R, t, pts[op[q]], p) > 0
    # without the v flip / frame turn the same data is far from the model
    bad = paper_F(cams, pts, oc, op, uv)
    assert bad > 1e6 * max(F0, 1e-30)


def test_intrinsics_series_reversion_order():
    # one camera, points at a shrinking field angle: the paper-model error of the converted camera falls like
    # |u|^7 when k1', k2' are right (ratio 2^7 per halving); a missing -2 k1^2 in k2' would leave |u|^5 (2^5)
    f, k1, k2 = 600.0, -0.25, 0.15
    cam = np.array([0, 0, 0, 0, 0, 0, f, k1, k2], float)

    def err_at(rho):
        X = np.array([[rho * 4.0, 0.0, -4.0]])              # BAL p = (rho, 0)
        u = B.bal_project(cam, X)
        c, uu = B.bal_to_paper(cam[None], u)
        n = oracle.bal_to_native(c)[0]
        return np.linalg.norm(oracle.reprojection_error(n[:9].reshape(3, 3), n[9:12], X[0], oracle.ray(n[12:], uu[0])))

    e = [err_at(0.08 / 2 ** s) for s in range(4)]
    ratios = [e[s] / e[s + 1] for s in range(3)]
    assert all(100 < q < 160 for q in ratios), ratios


def test_round_trip():
    r = np.random.default_rng(9)
    cams = np.hstack([Rotation.random(50, random_state=1).as_rotvec() * 0.99, r.normal(size=(50, 3)),
                      r.uniform(300, 900, (50, 1)), r.normal(size=(50, 2)) * 0.1])
    uv = r.normal(size=(20, 2)) * 100
    c, u = B.bal_to_paper(cams, uv)
    c2, u2 = B.paper_to_bal(c, u)
    np.testing.assert_array_equal(u2, uv)
    np.testing.assert_allclose(Rotation.from_rotvec(c2[:, :3]).as_matrix(), Rotation.from_rotvec(cams[:, :3]).as_matrix(),
                               atol=1e-14)
    np.testing.assert_allclose(c2[:, 3:], cams[:, 3:], rtol=1e-13, atol=1e-15)
