"""GPU parity of the NEXT-3 building block daba_coarse_blocks (include/daba.h) against oracle/coarse.normal_blocks:
the Gauss-Newton blocks of the intra-device penalties (readings R-N3a, R-N3b), element by element, fp64.

Tolerance: each block entry is a sum of O(100) products of O(1e6)-magnitude Jacobian entries evaluated in a
different order (FMA contraction on the GPU, none in the oracle), so entries are compared to 1e-11 relative to
the largest entry of their block (U, V, W, g) or of the sum (F)."""
import numpy as np
import pytest

import gen
import oracle
from oracle import coarse

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _blocks_gpu(cp, cams, pts, order, with_W=True):
    import paper_2305_07026_b200 as daba
    dev = torch.device("cuda:0")
    oc = cp.oc[order]
    cam_off = np.zeros(cp.M + 1, np.int64)
    np.add.at(cam_off, oc + 1, 1)
    cam_off = np.cumsum(cam_off)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
    out = daba.coarse_blocks(t(cams, torch.float64), t(pts, torch.float64), t(cp.op[order], torch.int32),
                             t(cp.uv[order], torch.float64), t(cam_off, torch.int64), loss=cp.opt.kind,
                             scale=cp.opt.scale, eps=cp.opt.eps, with_W=with_W)
    torch.cuda.synchronize()
    return [x.cpu().numpy() if x is not None else None for x in out]


def _close(gpu, ref, rel=1e-11):
    scale = np.abs(ref).reshape(ref.shape[0], -1).max(axis=1) if ref.ndim > 1 else np.abs(ref).max()
    scale = np.maximum(scale, 1e-300)
    err = np.abs(gpu - ref).reshape(ref.shape[0], -1).max(axis=1) if ref.ndim > 1 else np.abs(gpu - ref).max()
    assert np.all(err <= rel * scale), float(np.max(err / scale))


def _check(cp, cams, pts):
    order = np.argsort(cp.oc, kind="stable")
    U, gc, V, gl, W, Fc = coarse.normal_blocks(cp, cams, pts)
    gU, ggc, gV, ggl, gW, gF = _blocks_gpu(cp, cams, pts, order)
    _close(gU, U)
    _close(ggc, gc)
    _close(gV, V)
    _close(ggl, gl)
    _close(gW, W[order])
    assert gF.sum() == pytest.approx(Fc.sum(), rel=1e-12)
    _close(gF, Fc)
    # without W: U, g_c and the point blocks from the structure of J_c (the path of daba_coarse_run)
    sU, sgc, sV, sgl, sW, sF = _blocks_gpu(cp, cams, pts, order, with_W=False)
    assert sW is None
    _close(sU, U)
    _close(sgc, gc)
    _close(sV, V)
    _close(sgl, gl)
    _close(sF, Fc)


@pytest.mark.parametrize("loss", [oracle.LOSS_TRIVIAL, oracle.LOSS_HUBER, oracle.LOSS_CAUCHY])
def test_coarse_blocks_tiny(loss):
    p = gen.generate("tiny_seq", loss=loss, outlier_frac=0.05 if loss else 0.0)
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int))
    _check(cp, cp.cams0, cp.pts0)


def test_coarse_blocks_many_ctas_shuffled_order():
    # 3001 observations over 29 cameras (~100 per camera and more: up to several strides of the 128-thread CTA),
    # observations in a shuffled order (sorted by camera here, as the ABI requires; W compared in that order)
    p = gen.generate("small_cauchy", K=3001, N=700, M=29)
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int))
    perm = np.random.default_rng(1).permutation(cp.K)
    cp.oc, cp.op, cp.uv = cp.oc[perm], cp.op[perm], cp.uv[perm]
    _check(cp, cp.cams0, cp.pts0)


def test_coarse_blocks_degenerate_pair_and_empty_camera():
    p = gen.generate("tiny_seq", loss=oracle.LOSS_HUBER)
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int))
    pts = cp.pts0.copy()
    k0 = 5
    pts[cp.op[k0]] = cp.cams0[cp.oc[k0], 9:12]  # Assumption 2 fails for every pair of that point and camera
    # camera 0 loses its observations (moved to camera 1): an empty segment
    cp.oc = np.where(cp.oc == 0, 1, cp.oc)
    _check(cp, cp.cams0, pts)


def test_coarse_blocks_no_observations():
    import paper_2305_07026_b200 as daba
    dev = torch.device("cuda:0")
    cams = torch.zeros((3, 15), dtype=torch.float64, device=dev)
    pts = torch.ones((2, 3), dtype=torch.float64, device=dev)
    U, gc, V, gl, W, F = daba.coarse_blocks(cams, pts, torch.zeros(0, dtype=torch.int32, device=dev),
                                            torch.zeros((0, 2), dtype=torch.float64, device=dev),
                                            torch.zeros(4, dtype=torch.int64, device=dev))
    torch.cuda.synchronize()
    assert W.shape == (0, 9, 3)
    for x in (U, gc, V, gl, F):
        assert torch.count_nonzero(x).item() == 0


def _solve_gpu(cp, cams, pts, mu, max_iter=2000, tol=1e-15):
    import paper_2305_07026_b200 as daba
    dev = torch.device("cuda:0")
    order = np.argsort(cp.oc, kind="stable")
    cam_off = np.concatenate([[0], np.cumsum(np.bincount(cp.oc, minlength=cp.M))]).astype(np.int64)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
    oc, op, off = t(cp.oc[order], torch.int32), t(cp.op[order], torch.int32), t(cam_off, torch.int64)
    blocks = daba.coarse_blocks(t(cams, torch.float64), t(pts, torch.float64), op, t(cp.uv[order], torch.float64),
                                off, loss=cp.opt.kind, scale=cp.opt.scale, eps=cp.opt.eps)
    dc, dl, info = daba.coarse_solve(blocks, oc, op, off, xi=cp.opt.xi, mu=mu, max_iter=max_iter, tol=tol)
    torch.cuda.synchronize()
    return dc.cpu().numpy(), dl.cpu().numpy(), info


@pytest.mark.parametrize("cfg,loss,mu", [("tiny_seq", oracle.LOSS_TRIVIAL, 1e-3), ("tiny_seq", oracle.LOSS_HUBER, 1e-2),
                                         ("small", oracle.LOSS_CAUCHY, 1e-3)])
def test_coarse_solve_is_the_dense_lm_direction(cfg, loss, mu):
    """The Schur-complement PCG direction equals the oracle's dense Jacobi-scaled Cholesky solve of the same damped
    system (one device: every pair intra-device).  Tolerance 1e-7 of the largest entry: the PCG stops at a
    preconditioned residual ratio of 1e-15 on a system whose gauge directions only the proximal term xi = 1e-4 and
    the damping fix (condition ~1e8)."""
    p = (gen.generate("small_cauchy", K=3001, N=700, M=29) if cfg == "small"
         else gen.generate(cfg, loss=loss, outlier_frac=0.05 if loss else 0.0))
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int))
    H, g, ci, pj, cpos, ppos = cp.device_system(0, cp.cams0, cp.pts0)
    ref = coarse.Problem.lm_direction(H, g, mu)
    rc, rl = ref[:9 * p.M].reshape(p.M, 9), ref[9 * p.M:].reshape(p.N, 3)
    dc, dl, (iters, res) = _solve_gpu(cp, cp.cams0, cp.pts0, mu)
    assert iters >= 1
    ec = np.abs(dc - rc).max() / np.abs(rc).max()
    el = np.abs(dl - rl).max() / np.abs(rl).max()
    assert ec <= 1e-7 and el <= 1e-7, (ec, el, iters, res)


@pytest.mark.parametrize("loss,eta", [(oracle.LOSS_TRIVIAL, 0.1), (oracle.LOSS_HUBER, 1.0), (oracle.LOSS_CAUCHY, 0.1)])
def test_coarse_run_one_device_matches_the_oracle(loss, eta):
    """daba_coarse_run (Algorithm 1, coarse surrogate, one device) against oracle/coarse.run on the same inputs:
    restart flags identical, F / F-bar / E traces within 1e-9 relative, states within 1e-7 of their scale after 8
    iterations (the PCG direction agrees with the dense solve to ~1e-10, which the iteration carries along)."""
    import paper_2305_07026_b200 as daba
    p = gen.generate("tiny_seq", loss=loss, outlier_frac=0.05 if loss else 0.0)
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int), eta=eta)
    tr_ref, c_ref, l_ref = coarse.run(cp, 8)
    dev = torch.device("cuda:0")
    order = np.argsort(cp.oc, kind="stable")
    cam_off = np.concatenate([[0], np.cumsum(np.bincount(cp.oc, minlength=cp.M))]).astype(np.int64)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
    cams, pts = t(cp.cams0, torch.float64), t(cp.pts0, torch.float64)
    tr = daba.coarse_run(cams, pts, t(cp.oc[order], torch.int32), t(cp.op[order], torch.int32),
                         t(cp.uv[order], torch.float64), t(cam_off, torch.int64), 8, loss=cp.opt.kind,
                         scale=cp.opt.scale, xi=cp.opt.xi, eta=eta, pcg_max_iter=2000, pcg_tol=1e-15)
    np.testing.assert_array_equal(tr[:, 3], tr_ref[:, 3])
    for col in (0, 1, 2, 4):
        np.testing.assert_allclose(tr[:, col], tr_ref[:, col], rtol=1e-9)
    c, l = cams.cpu().numpy(), pts.cpu().numpy()
    assert np.abs(c - c_ref).max() <= 1e-7 * np.abs(c_ref).max()
    assert np.abs(l - l_ref).max() <= 1e-7 * np.abs(l_ref).max()
    assert tr[-1, 0] < tr[0, 0]


@pytest.mark.parametrize("eta", [0.1, 1.0])
def test_coarse_run_inexact_solve_keeps_the_mm_invariants(eta):
    """The timed configuration (PCG capped at a few iterations) is a different, inexact iterate sequence, so it is
    checked by what holds for any accepted LM step: E(x_mm | x^k) <= F(x^k) (accepted only on a decrease),
    E(x_acc | x^k) <= F-bar^k when not restarted (Alg. 1), and F(x^{k+1}) <= E(x^{k+1} | x^k) (Prop. 2)."""
    import paper_2305_07026_b200 as daba
    p = gen.generate("small_cauchy", K=3001, N=700, M=29)
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int))
    dev = torch.device("cuda:0")
    order = np.argsort(cp.oc, kind="stable")
    cam_off = np.concatenate([[0], np.cumsum(np.bincount(cp.oc, minlength=cp.M))]).astype(np.int64)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
    cams, pts = t(cp.cams0, torch.float64), t(cp.pts0, torch.float64)
    tr = daba.coarse_run(cams, pts, t(cp.oc[order], torch.int32), t(cp.op[order], torch.int32),
                         t(cp.uv[order], torch.float64), t(cam_off, torch.int64), 12, loss=cp.opt.kind,
                         scale=cp.opt.scale, eta=eta, pcg_max_iter=3, pcg_tol=1e-2)
    F, Fbar, Eacc, rs, Emm = tr.T
    rel = 1e-12
    assert np.all(Emm <= F * (1 + rel))
    assert np.all(Eacc[rs == 0] <= Fbar[rs == 0] * (1 + rel))
    Esel = np.where(rs == 1, Emm, Eacc)
    assert np.all(F[1:] <= Esel[:-1] * (1 + rel))
    assert F[-1] < F[0]


def test_coarse_run_isolated_camera_and_point():
    """A camera and a point without observations (degenerate cases of the method): their gradient is zero and only
    the proximal term acts on them, so they do not move (beyond ProjRot3D's rounding), and the rest of the run is
    the run without them."""
    import paper_2305_07026_b200 as daba
    p = gen.generate("tiny_seq", loss=oracle.LOSS_HUBER, outlier_frac=0.05)
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int))
    dev = torch.device("cuda:0")
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
    order = np.argsort(cp.oc, kind="stable")

    def run(cams0, pts0, M):
        off = np.concatenate([[0], np.cumsum(np.bincount(cp.oc, minlength=M))]).astype(np.int64)
        c, l = t(cams0, torch.float64), t(pts0, torch.float64)
        tr = daba.coarse_run(c, l, t(cp.oc[order], torch.int32), t(cp.op[order], torch.int32),
                             t(cp.uv[order], torch.float64), t(off, torch.int64), 5, loss=cp.opt.kind,
                             scale=cp.opt.scale, pcg_max_iter=2000, pcg_tol=1e-15)
        return tr, c.cpu().numpy(), l.cpu().numpy()

    tr0, c0, l0 = run(cp.cams0, cp.pts0, cp.M)
    extra_cam = cp.cams0[:1].copy()
    extra_cam[0, 9:12] += 3.0
    cams = np.vstack([cp.cams0, extra_cam])
    pts = np.vstack([cp.pts0, [[1.0, 2.0, 3.0]]])
    tr1, c1, l1 = run(cams, pts, cp.M + 1)
    np.testing.assert_array_equal(tr1[:, 3], tr0[:, 3])
    np.testing.assert_allclose(tr1[:, [0, 1, 2, 4]], tr0[:, [0, 1, 2, 4]], rtol=1e-11)
    np.testing.assert_allclose(c1[:-1], c0, rtol=0, atol=1e-9 * np.abs(c0).max())
    np.testing.assert_allclose(l1[:-1], l0, rtol=0, atol=1e-9 * np.abs(l0).max())
    # unchanged up to the rounding of ProjRot3D in the extrapolation (x-bar of a variable with x^k = x^{k-1})
    np.testing.assert_allclose(c1[-1], cams[-1], rtol=0, atol=1e-13 * np.abs(cams[-1]).max())
    np.testing.assert_array_equal(l1[-1], pts[-1])


# ---------------------------------------------------------------- NEXT-3 over a device partition
def _run_part_gpu(cp, iters, cam_dev=None, pt_dev=None, **opts):
    import paper_2305_07026_b200 as daba
    dev = torch.device("cuda:0")
    order = np.argsort(cp.oc, kind="stable")
    cam_off = np.concatenate([[0], np.cumsum(np.bincount(cp.oc, minlength=cp.M))]).astype(np.int64)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
    cams, pts = t(cp.cams0, torch.float64), t(cp.pts0, torch.float64)
    cd = t(cam_dev, torch.int32) if cam_dev is not None else None
    pd = t(pt_dev, torch.int32) if pt_dev is not None else None
    kw = dict(loss=cp.opt.kind, scale=cp.opt.scale, xi=cp.opt.xi, eta=cp.opt.eta, pcg_max_iter=2000, pcg_tol=1e-15,
              mm_always=1)
    kw.update(opts)
    tr, trials = daba.coarse_run_part(cams, pts, t(cp.oc[order], torch.int32), t(cp.op[order], torch.int32),
                                      t(cp.uv[order], torch.float64), t(cam_off, torch.int64), iters, cam_dev=cd,
                                      pt_dev=pd, **kw)
    return tr, trials, cams.cpu().numpy(), pts.cpu().numpy()


def _partition(p, ndev, kind, seed=0):
    rng = np.random.default_rng(seed)
    if kind == "random":
        return rng.integers(0, ndev, p.M), rng.integers(0, ndev, p.N)
    # contiguous camera ranges; each point with the device owning most of its observations (ties: lowest)
    cam_dev = (np.arange(p.M) * ndev) // p.M
    cnt = np.zeros((p.N, ndev), int)
    np.add.at(cnt, (p.obs_pt, cam_dev[p.obs_cam]), 1)
    return cam_dev, cnt.argmax(axis=1)


@pytest.mark.parametrize("ndev,kind,loss,eta,det", [(2, "contiguous", oracle.LOSS_HUBER, 0.1, 0),
                                                    (3, "random", oracle.LOSS_CAUCHY, 1.0, 1),
                                                    (2, "random", oracle.LOSS_TRIVIAL, 1.0, 0),
                                                    (2, "contiguous", oracle.LOSS_HUBER, 0.1, 1)])
def test_coarse_run_partitioned_matches_the_oracle(ndev, kind, loss, eta, det):
    """daba_coarse_run_part (eq. Ealpha: E' pairs exact in their device's LM step, E'' pairs majorized by P on the
    camera's device and Q on the point's; each device accepts its own first decreasing trial) against
    oracle/coarse.run with the same device assignment: restart flags identical, F / F-bar / E traces within 1e-9,
    states within 1e-7 of their scale after 8 iterations."""
    p = gen.generate("tiny_seq", loss=loss, outlier_frac=0.05 if loss else 0.0)
    cam_dev, pt_dev = _partition(p, ndev, kind, seed=ndev)
    cp = coarse.Problem(p, cam_dev, pt_dev, eta=eta)
    assert 0 < cp.intra.sum() < cp.K  # both kinds of pairs occur
    tr_ref, c_ref, l_ref = coarse.run(cp, 8)
    tr, trials, c, l = _run_part_gpu(cp, 8, cam_dev, pt_dev, deterministic=det)
    np.testing.assert_array_equal(tr[:, 3], tr_ref[:, 3])
    for col in (0, 1, 2, 4):
        np.testing.assert_allclose(tr[:, col], tr_ref[:, col], rtol=1e-9)
    assert np.abs(c - c_ref).max() <= 1e-7 * np.abs(c_ref).max()
    assert np.abs(l - l_ref).max() <= 1e-7 * np.abs(l_ref).max()
    assert trials.shape == (8, 2, ndev) and (trials[:, 1] >= 0).any()
    assert tr[-1, 0] < tr[0, 0]


def test_coarse_run_one_device_entries_agree():
    """daba_coarse_run is daba_coarse_run_part with one device (mm_always = 1)."""
    import paper_2305_07026_b200 as daba
    p = gen.generate("tiny_seq", loss=oracle.LOSS_HUBER, outlier_frac=0.05)
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int))
    tr1, _, c1, l1 = _run_part_gpu(cp, 6)
    dev = torch.device("cuda:0")
    order = np.argsort(cp.oc, kind="stable")
    cam_off = np.concatenate([[0], np.cumsum(np.bincount(cp.oc, minlength=cp.M))]).astype(np.int64)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
    cams, pts = t(cp.cams0, torch.float64), t(cp.pts0, torch.float64)
    tr0 = daba.coarse_run(cams, pts, t(cp.oc[order], torch.int32), t(cp.op[order], torch.int32),
                          t(cp.uv[order], torch.float64), t(cam_off, torch.int64), 6, loss=cp.opt.kind,
                          scale=cp.opt.scale, pcg_max_iter=2000, pcg_tol=1e-15)
    # (the point sums with fp64 atomics: two runs agree to rounding, not bitwise — include/daba.h)
    np.testing.assert_array_equal(tr1[:, 3], tr0[:, 3])
    np.testing.assert_allclose(tr1, tr0, rtol=1e-10)
    np.testing.assert_allclose(c1, cams.cpu().numpy(), rtol=0, atol=1e-10 * np.abs(c1).max())


@pytest.mark.parametrize("ndev", [1, 2])
def test_coarse_run_mm_only_on_restart(ndev):
    """mm_always = 0 solves the MM subproblem only when the restart fires (Alg. 1): the same iterates as
    solving it every iteration, E(x_mm | x^k) reported only on restarts."""
    p = gen.generate("tiny_seq", loss=oracle.LOSS_HUBER, outlier_frac=0.05)
    cam_dev, pt_dev = _partition(p, ndev, "contiguous")
    cp = coarse.Problem(p, cam_dev, pt_dev, eta=1.0)
    kw = dict(cam_dev=cam_dev, pt_dev=pt_dev) if ndev > 1 else {}
    tra, _, ca, la = _run_part_gpu(cp, 10, mm_always=1, deterministic=1, **kw)
    trb, trials_b, cb, lb = _run_part_gpu(cp, 10, mm_always=0, deterministic=1, **kw)
    rs = tra[:, 3] == 1
    assert rs.any() and (~rs).any()
    np.testing.assert_array_equal(trb[:, :4], tra[:, :4])  # (deterministic mode: bit for bit)
    np.testing.assert_array_equal(trb[rs, 4], tra[rs, 4])
    assert np.all(np.isnan(trb[~rs, 4])) and np.all(trials_b[~rs, 1] == -1)
    np.testing.assert_array_equal(cb, ca)
    np.testing.assert_array_equal(lb, la)


@pytest.mark.parametrize("ndev", [1, 3])
def test_coarse_run_deterministic_mode(ndev):
    """deterministic = 1 takes every sum in a fixed order (the point sides over a stable sort by point, the PCG
    scalars by per-CTA partials; no fp64 atomics): two runs of the inexact configuration the timing tools use (PCG
    <= 3 iterations, tol 1e-1) give identical traces, accepted trials and states; and they equal the atomic mode's
    run to rounding (the same iteration, another summation order)."""
    p = gen.generate("ladybug49", loss=oracle.LOSS_HUBER, outlier_frac=0.05)
    cam_dev, pt_dev = _partition(p, ndev, "contiguous")
    cp = coarse.Problem(p, cam_dev, pt_dev, eta=0.1)
    kw = dict(cam_dev=cam_dev, pt_dev=pt_dev) if ndev > 1 else {}
    runs = [_run_part_gpu(cp, 6, pcg_max_iter=3, pcg_tol=1e-1, mm_always=0, deterministic=1, **kw) for _ in range(2)]
    for a, b in zip(runs[0], runs[1]):
        np.testing.assert_array_equal(a, b)
    assert runs[0][0][-1, 0] < runs[0][0][0, 0]
    tr, trials, c, l = _run_part_gpu(cp, 6, pcg_max_iter=3, pcg_tol=1e-1, mm_always=0, **kw)
    np.testing.assert_array_equal(tr[:, 3], runs[0][0][:, 3])
    np.testing.assert_array_equal(trials, runs[0][1])
    np.testing.assert_allclose(tr[:, :3], runs[0][0][:, :3], rtol=1e-9)
    assert np.abs(c - runs[0][2]).max() <= 1e-7 * np.abs(c).max()
    assert np.abs(l - runs[0][3]).max() <= 1e-7 * np.abs(l).max()


def test_coarse_entries_reject_bad_indices_before_writing():
    """Index values are checked on the device before any kernel writes: an out-of-range point index, a camera
    segment table that does not end at K, a device id out of range -> DABA_E_INVALID_ARG, state untouched."""
    import paper_2305_07026_b200 as daba
    p = gen.generate("tiny_seq")
    cp = coarse.Problem(p, np.zeros(p.M, int), np.zeros(p.N, int))
    dev = torch.device("cuda:0")
    order = np.argsort(cp.oc, kind="stable")
    cam_off = np.concatenate([[0], np.cumsum(np.bincount(cp.oc, minlength=cp.M))]).astype(np.int64)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
    op_bad = cp.op[order].copy()
    op_bad[3] = cp.N
    off_bad = cam_off.copy()
    off_bad[-1] -= 1
    cases = [(op_bad, cam_off, None), (cp.op[order], off_bad, None),
             (cp.op[order], cam_off, (np.full(cp.M, 2), np.zeros(cp.N, int)))]
    for op, off, part in cases:
        cams, pts = t(cp.cams0, torch.float64), t(cp.pts0, torch.float64)
        kw = {}
        if part is not None:
            kw = dict(cam_dev=t(part[0], torch.int32), pt_dev=t(part[1], torch.int32), ndev=2)
        with pytest.raises(daba.DabaError) as e:
            daba.coarse_run_part(cams, pts, t(cp.oc[order], torch.int32), t(op, torch.int32),
                                 t(cp.uv[order], torch.float64), t(off, torch.int64), 2, **kw)
        assert e.value.code == -1
        np.testing.assert_array_equal(cams.cpu().numpy(), cp.cams0)
        np.testing.assert_array_equal(pts.cpu().numpy(), cp.pts0)
    with pytest.raises(daba.DabaError) as e:
        daba.coarse_blocks(t(cp.cams0, torch.float64), t(cp.pts0, torch.float64), t(op_bad, torch.int32),
                           t(cp.uv[order], torch.float64), t(cam_off, torch.int64))
    assert e.value.code == -1
    with pytest.raises(daba.DabaError):  # BAL-layout (M, 9) cameras: caught by the shape check
        daba.coarse_run_part(t(p.cams, torch.float64), t(cp.pts0, torch.float64), t(cp.oc[order], torch.int32),
                             t(cp.op[order], torch.int32), t(cp.uv[order], torch.float64), t(cam_off, torch.int64), 1)


@pytest.mark.parametrize("nranks,loss,eta,det", [(2, oracle.LOSS_HUBER, 0.1, 0), (3, oracle.LOSS_CAUCHY, 1.0, 1)])
def test_coarse_run_dist_matches_the_oracle(nranks, loss, eta, det):
    """NEXT-3 with one device per rank (daba_coarse_run_dist; ranks = threads through the LOCAL transport, each
    solving its own device's subproblem, allreducing F / E and exchanging the boundary variables): equal to
    oracle/coarse.run with the daba_create partition as the device assignment — restart flags identical, traces
    within 1e-9, every rank's owned states within 1e-7 of their scale after 8 iterations."""
    import threading
    import paper_2305_07026_b200 as daba
    p = gen.generate("tiny_seq", loss=loss, outlier_frac=0.05 if loss else 0.0)
    plan = daba.Plan(p.M, p.N, p.obs_cam, p.obs_pt, rank=0, nranks=nranks)
    cam_dev, pt_dev = plan.array(2), plan.array(3)
    cp = coarse.Problem(p, cam_dev, pt_dev, eta=eta)
    assert 0 < cp.intra.sum() < cp.K
    tr_ref, c_ref, l_ref = coarse.run(cp, 8)
    key = np.random.default_rng(nranks + 10).bytes(128)
    out, err = [None] * nranks, []

    def work(r):
        try:
            out[r] = daba.coarse_run_dist(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, 8, rank=r, nranks=nranks,
                                          comm_key=key, comm=daba.COMM_LOCAL, loss=loss, scale=p.loss_scale, eta=eta,
                                          pcg_max_iter=2000, pcg_tol=1e-15, mm_always=1, deterministic=det)
        except Exception as e:  # pragma: no cover
            err.append(e)
    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    [t.start() for t in th]
    [t.join() for t in th]
    if err:
        raise err[0]
    c, l = np.full_like(c_ref, np.nan), np.full_like(l_ref, np.nan)
    for tr, cr, lr in out:
        np.testing.assert_array_equal(tr, out[0][0])  # every rank reports the same global trace
        c[~np.isnan(cr[:, 0])] = cr[~np.isnan(cr[:, 0])]
        l[~np.isnan(lr[:, 0])] = lr[~np.isnan(lr[:, 0])]
    tr = out[0][0]
    np.testing.assert_array_equal(tr[:, 3], tr_ref[:, 3])
    for col in (0, 1, 2, 4):
        np.testing.assert_allclose(tr[:, col], tr_ref[:, col], rtol=1e-9)
    assert not np.isnan(c).any() and not np.isnan(l).any()
    assert np.abs(c - c_ref).max() <= 1e-7 * np.abs(c_ref).max()
    assert np.abs(l - l_ref).max() <= 1e-7 * np.abs(l_ref).max()
