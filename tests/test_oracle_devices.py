"""Pins for the oracle's decentralized adaptive restart (§5, eqs. DEalpha, Fainit, Fak, lFak, Eak;
Algorithm 1).

Fixed by what the paper and the mathematics imply, not by retyping the update:
  - one device is the global test (E'' is empty, F^{(k)} = F(x^k) by Lemma 1(a));
  - the per-device objectives add up to the objective: sum_a F^{a(k)} = F(x^k) for every partition (the kappa
    weights of eq. DEalpha split each pair's gap exactly once);
  - sum_a E^{a(k+1)} = E(x^{k+1} | x^k) of the mixed iterate, evaluated literally with eqs. P/Q, and it
    majorizes F(x^{k+1}) (Prop. 2);
  - a device that restarts has E^a_mm <= F^{a(k)} (the MM update decreases its surrogate); one that
    does not has E^a_acc <= F-bar^{a(k)} (Alg. 1);
  - on a noiseless problem F -> 0 under per-device restarts (Prop. amm).
"""
import numpy as np
import pytest

import gen
import oracle

XI = 1e-4


def owners(p, ndev, seed):
    """Random device ownership of cameras and points (every device non-empty)."""
    r = np.random.default_rng(seed)
    cd = r.integers(0, ndev, p.M).astype(np.int32)
    pd = r.integers(0, ndev, p.N).astype(np.int32)
    cd[:ndev] = np.arange(ndev)
    pd[:ndev] = np.arange(ndev)
    return cd, pd


def literal_E(p, ck, lk, c, l, sel_c=None, sel_l=None):
    """eq. Ealpha (D1) restricted to the selected variables: sum over the selected cameras of sum_j P_ij(c_i|x^k),
    over the selected points of sum_i Q_ij(l_j|x^k), plus xi/2 ||x - x^k||^2 over the selected variables."""
    sel_c = np.ones(p.M, bool) if sel_c is None else sel_c
    sel_l = np.ones(p.N, bool) if sel_l is None else sel_l
    tot = 0.0
    for k in range(p.K):
        i, j = p.obs_cam[k], p.obs_pt[k]
        coef = oracle.coefficients(ck[i], lk[j], p.obs_uv[k], p.loss, p.loss_scale)
        if sel_c[i]:
            tot += oracle.P(coef, c[i], p.obs_uv[k])
        if sel_l[j]:
            tot += oracle.Q(coef, l[j])
    return tot + 0.5 * XI * (np.sum((c - ck)[sel_c] ** 2) + np.sum((l - lk)[sel_l] ** 2))


@pytest.mark.parametrize("eta", [0.1, 1.0])
def test_single_device_is_the_global_test(eta):
    p = gen.generate("small_huber")
    a = oracle.Oracle(p, eta=eta)
    b = oracle.Oracle(p, eta=eta)
    b.set_devices(np.zeros(p.M, np.int32), np.zeros(p.N, np.int32))
    ta, tb = a.iterate(25), b.iterate(25)
    np.testing.assert_array_equal(ta[:, oracle.TR_RESTART], tb[:, oracle.TR_RESTART])
    for col in (oracle.TR_F, oracle.TR_FBAR, oracle.TR_EACC, oracle.TR_EMM):
        np.testing.assert_allclose(tb[:, col], ta[:, col], rtol=1e-11)
    ca, la = a.state(0)
    cb, lb = b.state(0)
    np.testing.assert_allclose(cb, ca, rtol=0, atol=1e-12)
    np.testing.assert_allclose(lb, la, rtol=1e-12)


@pytest.mark.parametrize("name,ndev,eta", [("small_huber", 2, 1.0), ("small_cauchy", 3, 0.1), ("tiny_seq", 3, 1.0)])
def test_device_objectives_add_up(name, ndev, eta):
    p = gen.generate(name)
    o = oracle.Oracle(p, eta=eta)
    cd, pd = owners(p, ndev, 5)
    o.set_devices(cd, pd)
    restarts = 0
    for k in range(20):
        tr = o.iterate(1)
        m = o.device_metrics()
        restarts += int(m[:, oracle.DEV_RESTART].sum())
        assert m[:, oracle.DEV_F].sum() == pytest.approx(tr[0, oracle.TR_F], rel=1e-10)
        # Alg. 1: a device keeps x_acc only if E_acc <= F-bar; after a restart its MM surrogate decreased
        for a in range(ndev):
            F, Fb, Ea, Em, r = m[a]
            if r:
                assert Em <= F + 1e-12 * abs(tr[0, oracle.TR_F])
            else:
                assert Ea <= Fb
    if eta == 1.0:
        assert restarts > 0  # the per-device tests actually fire


def test_mixed_iterate_surrogate_literal():
    # sum_a E^{a(k+1)} = E(x^{k+1} | x^k) (eq. Eak summed, with sum_a F^{a(k)} = F(x^k)), evaluated literally with
    # eqs. P/Q at the mixed iterate; per device, E^{a(k+1)} - F^{a(k)} = E^a(x^{a(k+1)}|x^k) - E^a(x^{a(k)}|x^k)
    p = gen.generate("tiny_seq")
    o = oracle.Oracle(p, eta=1.0)
    cd, pd = owners(p, 2, 11)
    o.set_devices(cd, pd)
    for k in range(8):
        ck, lk = o.state(0)
        tr = o.iterate(1)
        c1, l1 = o.state(0)
        m = o.device_metrics()
        E_sel = np.where(m[:, oracle.DEV_RESTART] > 0, m[:, oracle.DEV_EMM], m[:, oracle.DEV_EACC])
        E_lit = literal_E(p, ck, lk, c1, l1)
        assert E_sel.sum() == pytest.approx(E_lit, rel=1e-9)
        for a in range(2):
            da = literal_E(p, ck, lk, c1, l1, cd == a, pd == a) - literal_E(p, ck, lk, ck, lk, cd == a, pd == a)
            assert E_sel[a] - m[a, oracle.DEV_F] == pytest.approx(da, rel=1e-7, abs=1e-9 * tr[0, oracle.TR_F])
        # Prop. 2: the surrogate of the mixed iterate majorizes the objective there
        F1 = oracle.Oracle(gen.Problem(p.name, oracle.native_to_bal(c1), l1, p.obs_cam, p.obs_pt, p.obs_uv,
                                       p.gt_cams, p.gt_pts, p.loss, p.loss_scale)).objective()
        assert F1 + 0.5 * XI * (np.sum((c1 - ck) ** 2) + np.sum((l1 - lk) ** 2)) <= E_lit * (1 + 1e-12)


def test_convergence_with_device_restarts():
    # Prop. amm: with per-device restarts the iterates still converge; noiseless -> F -> 0
    p = gen.generate("tiny_seq", noise_px=0.0, outlier_frac=0.0)
    o = oracle.Oracle(p)
    cd, pd = owners(p, 3, 2)
    o.set_devices(cd, pd)
    tr = o.iterate(1500)
    F = tr[:, oracle.TR_F]
    assert F[-1] < 1e-5 * F[0]
