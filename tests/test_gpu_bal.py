"""GPU: the pixel reprojection metric (daba_pixel_error) against the oracle's BAL metric
(oracle/bal.py), and a BAL file solved end to end (native read -> convention map -> DABA iterations)."""
import threading

import numpy as np
import pytest

import gen
from oracle import bal as B
from test_oracle_bal import bal_scene

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2305_07026_b200")


def solver(cams, pts, oc, op, uv, **kw):
    return D.Solver(cams, pts, oc, op, uv, **kw)


def oracle_metric(cams_abi, pts, oc, op, uv_abi):
    cb, ub = B.paper_to_bal(cams_abi, uv_abi)
    return B.mean_pixel_error(cb, pts, oc, op, ub)


@pytest.mark.parametrize("name", ["tiny_seq", "small_huber", "ladybug49"])
def test_pixel_error_matches_oracle(name):
    p = gen.generate(name)
    with solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale) as s:
        for it in (0, 15):
            if it:
                s.iterate(it)
            g = s.pixel_error()
            cams, pts, _ = s.state()
            o = oracle_metric(cams, pts, p.obs_cam, p.obs_pt, p.obs_uv)
            assert g["count"] == o[3] == p.K
            assert g["behind"] == o[2]
            assert g["sum"] == pytest.approx(o[0], rel=1e-11)
            assert g["sum_sq"] == pytest.approx(o[1], rel=1e-11)


def test_pixel_error_ranks_add_up():
    p = gen.generate("small_huber")
    with solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv) as s:
        ref = s.pixel_error()
    R = 3
    key = np.random.default_rng(7).bytes(128)
    out = [None] * R

    def work(r):
        with solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, rank=r, nranks=R, comm_key=key,
                    comm=D.COMM_LOCAL) as s:
            out[r] = s.pixel_error()
    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert sum(o["count"] for o in out) == ref["count"]
    assert sum(o["sum"] for o in out) == pytest.approx(ref["sum"], rel=1e-12)
    assert sum(o["sum_sq"] for o in out) == pytest.approx(ref["sum_sq"], rel=1e-12)


def test_bal_file_end_to_end(tmp_path):
    # a distorted, noisy BAL scene written as a file; read natively, mapped to the paper's convention, solved
    cams, pts, oc, op, uv = bal_scene(M=12, N=400, seed=21, k1=-0.08, k2=0.01, noise=0.5)
    r = np.random.default_rng(1)
    init_pts = pts + r.normal(size=pts.shape) * 0.02
    path = str(tmp_path / "scene.txt")
    D.write_bal(path, D.BalProblem(cams, init_pts, oc, op, uv))
    b = D.read_bal(path)
    c, u = D.bal_to_paper(b.cams, b.obs_uv)
    o0 = B.mean_pixel_error(cams, init_pts, oc, op, uv)  # the oracle on the BAL data as written
    with solver(c, b.pts, b.obs_cam, b.obs_pt, u) as s:
        g0 = s.pixel_error()
        assert g0["sum"] == pytest.approx(o0[0], rel=1e-9)
        assert g0["behind"] == 0
        s.iterate(300)
        g1 = s.pixel_error()
        cs, ps, _ = s.state()
    o1 = oracle_metric(cs, ps, oc, op, u)
    assert g1["sum"] == pytest.approx(o1[0], rel=1e-10)
    noise_floor = float(np.mean(np.linalg.norm(uv - np.concatenate([B.bal_project(cams[i], pts) for i in range(12)]),
                                               axis=1)))
    assert g1["mean"] < 0.5 * g0["mean"]
    assert g1["mean"] < 1.2 * noise_floor


def test_pixel_error_edge_cases():
    p = gen.generate("tiny_seq")
    # no observations: zero sums (the reduction runs over zero chunks)
    with D.Solver(p.cams, p.pts, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 2))) as s:
        g = s.pixel_error()
        assert (g["count"], g["sum"], g["sum_sq"], g["behind"]) == (0, 0.0, 0.0, 0)
    # points mirrored through one of their cameras' centres land behind it: counted, still summed like the oracle
    pts = p.pts.copy()
    cam0 = p.obs_cam[0]
    from oracle import bal_to_native
    centre = bal_to_native(p.cams[cam0:cam0 + 1])[0, 9:12]
    flip = np.unique(p.obs_pt[p.obs_cam == cam0])[:5]
    pts[flip] = 2 * centre - pts[flip]
    with solver(p.cams, pts, p.obs_cam, p.obs_pt, p.obs_uv) as s:
        g = s.pixel_error()
    o = oracle_metric(p.cams, pts, p.obs_cam, p.obs_pt, p.obs_uv)
    assert g["behind"] == o[2] >= 5
    assert g["sum"] == pytest.approx(o[0], rel=1e-11)


@pytest.mark.parametrize("name", ["small_huber", "ladybug49"])
def test_pixel_residuals_match_oracle(name):
    p = gen.generate(name)
    with solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv) as s:
        s.iterate(5)
        r = s.pixel_residuals()
        g = s.pixel_error()
        cams, pts, _ = s.state()
    cb, ub = B.paper_to_bal(cams, p.obs_uv)
    o, behind = B.pixel_residuals(cb, pts, p.obs_cam, p.obs_pt, ub)
    np.testing.assert_allclose(r, o, rtol=1e-10, atol=1e-10)
    assert r.sum() == pytest.approx(g["sum"], rel=1e-12)


def test_pixel_residuals_unsorted_and_ranks():
    # a permuted observation order (full host plan) and 2 LOCAL ranks: entries land at their input index
    p = gen.generate("small_huber")
    perm = np.random.default_rng(5).permutation(p.K)
    oc, op, uv = p.obs_cam[perm], p.obs_pt[perm], p.obs_uv[perm]
    with solver(p.cams, p.pts, oc, op, uv) as s:
        ref = s.pixel_residuals()
    assert np.isfinite(ref).all()
    key = np.random.default_rng(8).bytes(128)
    out = [None] * 2

    def work(r):
        with solver(p.cams, p.pts, oc, op, uv, rank=r, nranks=2, comm_key=key, comm=D.COMM_LOCAL) as s:
            out[r] = s.pixel_residuals()
    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    have = [np.isfinite(o) for o in out]
    assert not (have[0] & have[1]).any() and (have[0] | have[1]).all()
    merged = np.where(have[0], out[0], out[1])
    np.testing.assert_allclose(merged, ref, rtol=1e-13)
