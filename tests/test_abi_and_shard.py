"""CPU tests of the boundary: libdaba.so loads and exports every symbol include/daba.h declares; the host-side
shard planner (P:L532 partition; halo lists of Alg. 1) is consistent across ranks — single process here,
and over gloo with world_size 2 (multiprocess) as the N > 1 path runs it."""
import os
import re
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import paper_2305_07026_b200 as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "daba.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(daba_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 20
    L = D.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(D.daba.EXPORTS) <= set(names)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2305_07026_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("no code shared with", ""), f


def check_plans(p, nranks):
    plans = [D.Plan(p.M, p.N, p.obs_cam, p.obs_pt, rank=r, nranks=nranks) for r in range(nranks)]
    cam_owner, pt_owner = plans[0].array(2), plans[0].array(3)
    # ownership is total and agreed by every rank
    for pl in plans[1:]:
        np.testing.assert_array_equal(pl.array(2), cam_owner)
        np.testing.assert_array_equal(pl.array(3), pt_owner)
    assert sum(pl.counts["own_cams"] for pl in plans) == p.M
    assert sum(pl.counts["own_pts"] for pl in plans) == p.N
    assert sum(pl.counts["cam_side_obs"] for pl in plans) == p.K
    assert sum(pl.counts["pt_side_obs"] for pl in plans) == p.K
    # contiguous, balanced camera ranges
    assert np.all(np.diff(cam_owner) >= 0)
    sides = [pl.counts["cam_side_obs"] for pl in plans]
    assert max(sides) <= 1.5 * p.K / nranks + np.bincount(p.obs_cam).max()
    # plurality point owner, ties to the lowest rank
    for j in np.random.default_rng(0).choice(p.N, 200, replace=False):
        owners = cam_owner[p.obs_cam[p.obs_pt == j]]
        cnt = np.bincount(owners, minlength=nranks)
        assert pt_owner[j] == int(np.argmax(cnt))
    # halo lists are symmetric: what a sends to b is what b expects from a, in the same order
    for a, pa in enumerate(plans):
        peers_a = list(pa.array(4))
        for qa, b in enumerate(peers_a):
            pb = plans[b]
            qb = list(pb.array(4)).index(a)
            np.testing.assert_array_equal(pa.peer_list(qa, 0), pb.peer_list(qb, 2))
            np.testing.assert_array_equal(pa.peer_list(qa, 1), pb.peer_list(qb, 3))
    # a crossing observation (i, j) makes camera i a halo on j's owner and point j a halo on i's owner
    for k in np.random.default_rng(1).choice(p.K, 300, replace=False):
        i, j = p.obs_cam[k], p.obs_pt[k]
        a, b = cam_owner[i], pt_owner[j]
        if a != b:
            assert i in set(plans[b].array(0)[plans[b].counts["own_cams"]:])
            assert j in set(plans[a].array(1)[plans[a].counts["own_pts"]:])
    return plans


@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
def test_plan_invariants(nranks):
    check_plans(gen.generate("small_seq_huber"), nranks)
    check_plans(gen.generate("small_cauchy"), nranks)


def test_plan_rejects_bad_input():
    p = gen.generate("tiny_seq")
    with pytest.raises(D.DabaError):
        D.Plan(p.M, p.N, p.obs_cam, np.where(np.arange(p.K) == 0, p.N + 1, p.obs_pt))
    with pytest.raises(D.DabaError):
        D.Plan(p.M, p.N, np.concatenate([p.obs_cam, p.obs_cam[:1]]), np.concatenate([p.obs_pt, p.obs_pt[:1]]))


# ---------------------------------------------------------------- gloo, world_size 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = gen.generate("small_seq_huber")
        pl = D.Plan(p.M, p.N, p.obs_cam, p.obs_pt, rank=rank, nranks=world)
        own_c, own_p = pl.counts["own_cams"], pl.counts["own_pts"]
        cam_g, pt_g = pl.array(0), pl.array(1)
        # local state: owned entries hold a value known to everyone (f(global id)), halo slots NaN
        f_cam = lambda g: np.stack([g * 1.0 + k for k in range(15)], axis=-1)
        f_pt = lambda g: np.stack([-(g * 1.0) - k for k in range(3)], axis=-1)
        cams = np.full((cam_g.size, 15), np.nan)
        pts = np.full((pt_g.size, 3), np.nan)
        cams[:own_c] = f_cam(cam_g[:own_c])
        pts[:own_p] = f_pt(pt_g[:own_p])
        g2l_c = {g: i for i, g in enumerate(cam_g)}
        g2l_p = {g: i for i, g in enumerate(pt_g)}
        # one halo exchange exactly as the engine packs it: per peer [cams x 15 | points x 3]
        reqs, bufs = [], []
        for q_, b in enumerate(pl.array(4)):
            sc, sp = pl.peer_list(q_, 0), pl.peer_list(q_, 1)
            send = np.concatenate([cams[[g2l_c[g] for g in sc]].ravel(), pts[[g2l_p[g] for g in sp]].ravel()])
            rc, rp = pl.peer_list(q_, 2), pl.peer_list(q_, 3)
            recv = torch.zeros(15 * rc.size + 3 * rp.size, dtype=torch.float64)
            reqs.append(dist.isend(torch.from_numpy(send), int(b)))
            reqs.append(dist.irecv(recv, int(b)))
            bufs.append((rc, rp, recv))
        for r in reqs:
            r.wait()
        for rc, rp, recv in bufs:
            v = recv.numpy()
            cams[[g2l_c[g] for g in rc]] = v[:15 * rc.size].reshape(-1, 15)
            pts[[g2l_p[g] for g in rp]] = v[15 * rc.size:].reshape(-1, 3)
        ok = (not np.isnan(cams).any()) and (not np.isnan(pts).any())
        ok = ok and np.array_equal(cams, f_cam(cam_g)) and np.array_equal(pts, f_pt(pt_g))
        # global counts through an allreduce (the restart sums travel the same way)
        t = torch.tensor([pl.counts["cam_side_obs"], pl.counts["pt_side_obs"], own_c, own_p], dtype=torch.float64)
        dist.all_reduce(t)
        ok = ok and t.tolist() == [p.K, p.K, p.M, p.N]
        q.put((rank, bool(ok), pl.counts))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_over_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    [pr.start() for pr in procs]
    res = [q.get(timeout=240) for _ in procs]
    [pr.join(timeout=60) for pr in procs]
    assert all(ok for _, ok, _ in res), res
    assert all(c["halo_pts"] > 0 and c["halo_cams"] > 0 for _, _, c in res)


def test_missing_extension_fails_loudly(tmp_path):
    # no CPU fallback: without libdaba.so the binding raises on first use
    import subprocess
    import sys
    env = dict(os.environ, DABA_LIB=str(tmp_path / "absent" / "libdaba.so"))
    code = ("import paper_2305_07026_b200 as D\n"
            "try:\n    D.lib()\nexcept ImportError as e:\n    print('raised', e)\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert "raised" in out.stdout and "missing" in out.stdout, out.stdout + out.stderr


def test_coarse_entry_points_reject_bad_arguments():
    """include/daba.h NEXT-3 calls: invalid sizes, NULL buffers and unknown losses return DABA_E_INVALID_ARG (-1)
    before any CUDA call (so this runs without a GPU)."""
    L = D.lib()
    dummy = np.zeros(64)
    p = dummy.ctypes.data
    # daba_coarse_blocks(cams, M, pts, N, obs_pt, obs_uv, cam_off, K, loss, scale, eps, U, gc, V, gl, W, F, stream)
    assert L.daba_coarse_blocks(p, -1, p, 1, p, p, p, 1, 0, 1.0, 1e-8, p, p, p, p, p, p, None) == -1
    assert L.daba_coarse_blocks(p, 1, p, 1, p, p, p, 1, 3, 1.0, 1e-8, p, p, p, p, p, p, None) == -1   # loss
    assert L.daba_coarse_blocks(p, 1, p, 1, p, p, p, 1, 0, 0.0, 1e-8, p, p, p, p, p, p, None) == -1   # scale
    assert L.daba_coarse_blocks(None, 1, p, 1, p, p, p, 1, 0, 1.0, 1e-8, p, p, p, p, p, p, None) == -1
    assert L.daba_coarse_blocks(p, 1, p, 1, None, p, p, 1, 0, 1.0, 1e-8, p, p, p, p, p, p, None) == -1
    assert L.daba_coarse_solve_workspace(-1, 0) == -1
    assert L.daba_coarse_solve_workspace(2, 3) > 0
    info = np.zeros(2)
    args = [p, p, p, p, p, p, p, p, 1, 1, 1, 1e-4, 1e-3, 10, 1e-12, p, p, p, info.ctypes.data, None]
    bad = list(args)
    bad[12] = -1.0  # mu
    assert L.daba_coarse_solve(*bad) == -1
    bad = list(args)
    bad[18] = None  # info
    assert L.daba_coarse_solve(*bad) == -1
    bad = list(args)
    bad[4] = None  # W with K > 0
    assert L.daba_coarse_solve(*bad) == -1
    # daba_coarse_run(cams, M, pts, N, oc, op, uv, off, K, loss, scale, eps, xi, eta, mu0, mu_up, trials, acc,
    #                 pcg_iter, pcg_tol, n_iters, trace, stream)
    run = [p, 1, p, 1, p, p, p, p, 1, 0, 1.0, 1e-8, 1e-4, 0.1, 1e-3, 10.0, 5, 1, 10, 1e-10, 1, None, None]
    for idx, v in ((12, 0.0), (13, 0.0), (13, 1.5), (15, 0.5), (16, 0), (18, 0), (20, -1), (9, 7)):
        bad = list(run)
        bad[idx] = v
        assert L.daba_coarse_run(*bad) == -1, idx
