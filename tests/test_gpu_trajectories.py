"""50-iteration GPU trajectories at the full-size configs against stored oracle trajectories.

The goldens (tests/golden/traj_<config>_eta<eta>.npz) are written by tools/oracle_trajectories.py, which calls only
gen/ and oracle/ (the single-threaded CPU oracle, 50 iterations of Algorithm 1).  The GPU runs the same
generated input free (no re-anchoring) and is held to BASELINE.json's bar: F(x^k) within 1e-10 relative every
iteration — and F-bar likewise; E(x_acc|x^k), E(x_mm|x^k) (eqs. lFak, Eak) within 1e-9 — identical
restart flags, and camera / point states within 1e-8 after 50 iterations on the stored sample.
"""
import glob
import os

import numpy as np
import pytest

import gen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

D = pytest.importorskip("paper_2305_07026_b200")

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "traj_*.npz")))
TR_F, TR_FBAR, TR_EACC, TR_RESTART, TR_EMM = 0, 1, 2, 3, 4  # oracle.TR_* = daba.TR_* columns


def case_id(path):
    return os.path.basename(path)[5:-4]


def state_errors(cg, lg, co, lo):
    eR = np.linalg.norm(cg[:, :9] - co[:, :9], axis=1).max(initial=0)
    et = (np.linalg.norm(cg[:, 9:12] - co[:, 9:12], axis=1) / np.maximum(1, np.linalg.norm(co[:, 9:12], axis=1))).max(initial=0)
    ed = (np.linalg.norm(cg[:, 12:] - co[:, 12:], axis=1) / np.linalg.norm(co[:, 12:], axis=1)).max(initial=0)
    el = (np.linalg.norm(lg - lo, axis=1) / np.maximum(1, np.linalg.norm(lo, axis=1))).max(initial=0)
    return eR, et, ed, el


@pytest.mark.parametrize("path", GOLD, ids=[case_id(g) for g in GOLD])
def test_fifty_iterations_full_size(path):
    g = np.load(path)
    name, eta, iters = str(g["config"]), float(g["eta"]), int(g["iterations"])
    p = gen.generate(name)
    assert (p.M, p.N, p.K) == (int(g["M"]), int(g["N"]), int(g["K"]))
    tro = g["trace"]
    with D.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale, eta=eta) as s:
        assert s.objective() == pytest.approx(float(g["F0"]), rel=1e-10)
        trg = s.iterate_trace(iters)
        cg, lg, _ = s.state_native(0)
    # F(x^k) and F-bar at the north star's 1e-10.  E(x_acc|x^k) and E(x_mm|x^k) are surrogate values at the
    # candidates, not at the iterate: at an overshooting accelerated step (gamma ~ 0.9, restart fires, E_acc ~ 2 F)
    # they amplify the free-running trajectories' 1e-14-level state differences — Trafalgar eta = 0.1, k = 34:
    # 1.4e-10 free-running, 4e-16 when the oracle is re-anchored at the GPU's state
    # (profiles/r02_traj_diag_trafalgar_eta0.1_k34.log, tools/diag_trajectory.py) — so they are held to 1e-9
    # (reading R-T1).
    for col, tol in ((TR_F, 1e-10), (TR_FBAR, 1e-10), (TR_EACC, 1e-9), (TR_EMM, 1e-9)):
        rel = np.abs(trg[:, col] - tro[:, col]) / np.abs(tro[:, col])
        assert rel.max() <= tol, (col, rel.max(), int(rel.argmax()))
    np.testing.assert_array_equal(trg[:, TR_RESTART], tro[:, TR_RESTART])
    errs = state_errors(cg[g["cam_ids"]], lg[g["pt_ids"]], g["cams"], g["pts"])
    assert max(errs) <= 1e-8, errs
