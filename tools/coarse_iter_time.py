"""ms per NEXT-3 coarse iteration (daba_coarse_run_part, PCG <= 3 to 1e-1, MM only on restart) and F after n
iterations, for comparing builds (DABA_LIB=...).

    python tools/coarse_iter_time.py CONFIG N_ITERS NDEV
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

cfg = sys.argv[1] if len(sys.argv) > 1 else "final13682"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nd = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = gen.generate(cfg)
order, off = camera_sorted(p)
dev = torch.device("cuda:0")
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
args = (t(np.asarray(p.obs_cam)[order], torch.int32), t(np.asarray(p.obs_pt)[order], torch.int32),
        t(np.asarray(p.obs_uv).reshape(-1, 2)[order], torch.float64), t(off, torch.int64))
c0, l0 = t(bal_to_native(p.cams), torch.float64), t(np.asarray(p.pts).reshape(-1, 3), torch.float64)
kw = dict(loss=p.loss, scale=p.loss_scale, pcg_max_iter=3, pcg_tol=1e-1, mm_always=0, keep_scratch=1,
          deterministic=int(os.environ.get("COARSE_DET", "0")))
part = {}
if nd > 1:
    cd, pd = contiguous_partition(p, nd)
    part = dict(cam_dev=t(cd, torch.int32), pt_dev=t(pd, torch.int32), ndev=nd)
daba.coarse_run_part(c0.clone(), l0.clone(), *args, 1, **part, **kw)
res = []
for rep in range(2):
    cams, pts = c0.clone(), l0.clone()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    daba.coarse_run_part(cams, pts, *args, 1, **part, **kw)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tr, _ = daba.coarse_run_part(cams, pts, *args, n, **part, **kw)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    res.append(1e3 * (t3 - t2) / n)
print(json.dumps({"lib": os.environ.get("DABA_LIB", "default"), "config": cfg, "ndev": nd, "iters": n,
                  "ms_per_iter": min(res), "F": float(tr[-1, 0])}))
