"""NEXT-3 measurement: daba_coarse_run (coarse surrogate, one device, one successful Schur/PCG LM step per
subproblem) against the finest-partition production path (daba_iterate) on the same synthetic problem:
time per iteration and F after n iterations.  Usage: coarse_run_time.py CONFIG N_ITERS PCG_ITERS PCG_TOL"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402
from tools.coarse_common import bal_to_native, camera_sorted  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "venice1778_1m"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pcg = int(sys.argv[3]) if len(sys.argv) > 3 else 10
tol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-2
p = gen.generate(cfg)
order, off = camera_sorted(p)
dev = torch.device("cuda:0")
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
args = (t(np.asarray(p.obs_cam)[order], torch.int32), t(np.asarray(p.obs_pt)[order], torch.int32),
        t(np.asarray(p.obs_uv).reshape(-1, 2)[order], torch.float64), t(off, torch.int64))
res = {"config": cfg, "M": p.M, "N": p.N, "K": p.K, "loss": p.loss, "iters": n, "pcg_max_iter": pcg, "pcg_tol": tol}
# warm-up (one iteration on a copy), then the timed run
c0, l0 = t(bal_to_native(p.cams), torch.float64), t(np.asarray(p.pts).reshape(-1, 3), torch.float64)
daba.coarse_run(c0.clone(), l0.clone(), *args, 1, loss=p.loss, scale=p.loss_scale, pcg_max_iter=pcg, pcg_tol=tol)
cams, pts = c0.clone(), l0.clone()
torch.cuda.synchronize()
t0 = time.perf_counter()
tr = daba.coarse_run(cams, pts, *args, n, loss=p.loss, scale=p.loss_scale, pcg_max_iter=pcg, pcg_tol=tol)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
res["coarse"] = {"ms_per_iter": 1e3 * dt / n, "F": tr[:, 0].tolist() + [None], "restarts": int(tr[:, 3].sum())}
s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale)
Ff = [s.objective()]
for _ in range(n):
    s.iterate(1)
    Ff.append(s.objective())
s.close()
s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale)
s.iterate(3)
torch.cuda.synchronize()
t0 = time.perf_counter()
s.iterate(50)
s.objective()
res["finest"] = {"ms_per_iter": 1e3 * (time.perf_counter() - t0) / 50, "F": Ff}
# F after the coarse run's last iterate
s2 = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale)
s2.close()
s.close()
F_end = float(daba.coarse_blocks(cams, pts, args[1], args[2], args[3], loss=p.loss, scale=p.loss_scale)[5].sum())
res["coarse"]["F"][-1] = F_end
res["coarse"]["time_s"] = n * res["coarse"]["ms_per_iter"] / 1e3
# time to the coarse run's final accuracy on the finest partition: first k with F(x^k) <= F_end
s3 = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale)
cap = int(os.environ.get("FINEST_CAP", "3000"))
Ftr, _ = s3.iterate(cap, F_trace=True)
s3.close()
hit = np.flatnonzero(np.asarray(Ftr) <= F_end)
k = int(hit[0]) if hit.size else None
res["finest"]["iters_to_coarse_F"] = k
res["finest"]["time_s_to_coarse_F"] = None if k is None else k * res["finest"]["ms_per_iter"] / 1e3
print(json.dumps(res))
