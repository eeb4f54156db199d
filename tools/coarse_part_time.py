"""NEXT-3 over a device partition (daba_coarse_run_part, all devices on one GPU): time per iteration and F after n
iterations for ndev devices (contiguous camera ranges, plurality points), the MM subproblem only on restarts
(mm_always = 0), against the finest partition (daba_iterate) to the same F.

    python tools/coarse_part_time.py CONFIG N_ITERS PCG_ITERS PCG_TOL NDEV[,NDEV...]     (COARSE_DET=1: deterministic)
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402
from tools.coarse_common import bal_to_native, camera_sorted, contiguous_partition  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "venice1778_1m"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pcg = int(sys.argv[3]) if len(sys.argv) > 3 else 10
tol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-2
ndevs = [int(x) for x in (sys.argv[5] if len(sys.argv) > 5 else "1,2,4,8").split(",")]
p = gen.generate(cfg)
order, off = camera_sorted(p)
dev = torch.device("cuda:0")
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
args = (t(np.asarray(p.obs_cam)[order], torch.int32), t(np.asarray(p.obs_pt)[order], torch.int32),
        t(np.asarray(p.obs_uv).reshape(-1, 2)[order], torch.float64), t(off, torch.int64))
c0, l0 = t(bal_to_native(p.cams), torch.float64), t(np.asarray(p.pts).reshape(-1, 3), torch.float64)
# finest partition: F trace and time per iteration
s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale)
cap = int(os.environ.get("FINEST_CAP", "3000"))
Ftr, _ = s.iterate(cap, F_trace=True)
s.close()
s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale)
s.iterate(3)
s.objective()
t0 = time.perf_counter()
s.iterate(50)
s.objective()
finest_ms = 1e3 * (time.perf_counter() - t0) / 50
s.close()
out = {"config": cfg, "M": p.M, "N": p.N, "K": p.K, "iters": n, "pcg_max_iter": pcg, "pcg_tol": tol,
       "finest_ms_per_iter": finest_ms, "runs": []}
for nd in ndevs:
    cd, pd = contiguous_partition(p, nd)
    kw = dict(loss=p.loss, scale=p.loss_scale, pcg_max_iter=pcg, pcg_tol=tol, mm_always=0, keep_scratch=1,
              deterministic=int(os.environ.get("COARSE_DET", "0")))
    part = dict(cam_dev=t(cd, torch.int32), pt_dev=t(pd, torch.int32), ndev=nd) if nd > 1 else {}
    daba.coarse_run_part(c0.clone(), l0.clone(), *args, 1, **part, **kw)  # warm-up
    dt = float("inf")
    for rep in range(2):  # the faster of two runs (clocks vary under the power cap after the finest runs)
        cams, pts = c0.clone(), l0.clone()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr, trials = daba.coarse_run_part(cams, pts, *args, n, **part, **kw)
        torch.cuda.synchronize()
        dt = min(dt, time.perf_counter() - t0)
    F_end = float(daba.coarse_blocks(cams, pts, args[1], args[2], args[3], loss=p.loss, scale=p.loss_scale)[5].sum())
    hit = np.flatnonzero(np.asarray(Ftr) <= F_end)
    k = int(hit[0]) if hit.size else None
    intra = float(np.mean(cd[p.obs_cam] == pd[p.obs_pt]))
    out["runs"].append({"ndev": nd, "intra_pair_frac": round(intra, 4), "ms_per_iter": 1e3 * dt / n,
                        "F": [float(x) for x in tr[:, 0]] + [F_end], "restarts": int(tr[:, 3].sum()),
                        "finest_iters_to_F": k,
                        "finest_time_s_to_F": None if k is None else k * finest_ms / 1e3, "coarse_time_s": dt})
    print(json.dumps(out["runs"][-1]), flush=True)
print(json.dumps(out))
