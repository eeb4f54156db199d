"""A short NEXT-3 run for ncu (daba_coarse_run_part, PCG capped, MM only on restart)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402
from tools.coarse_common import bal_to_native, camera_sorted, contiguous_partition  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "final13682"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ndev = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = gen.generate(cfg)
order, off = camera_sorted(p)
dev = torch.device("cuda:0")
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
args = (t(np.asarray(p.obs_cam)[order], torch.int32), t(np.asarray(p.obs_pt)[order], torch.int32),
        t(np.asarray(p.obs_uv).reshape(-1, 2)[order], torch.float64), t(off, torch.int64))
cams, pts = t(bal_to_native(p.cams), torch.float64), t(np.asarray(p.pts).reshape(-1, 3), torch.float64)
part = {}
if ndev > 1:
    cd, pd = contiguous_partition(p, ndev)
    part = dict(cam_dev=t(cd, torch.int32), pt_dev=t(pd, torch.int32), ndev=ndev)
tr, _ = daba.coarse_run_part(cams, pts, *args, iters, loss=p.loss, scale=p.loss_scale, pcg_max_iter=3, pcg_tol=1e-1,
                             mm_always=0, deterministic=int(os.environ.get("COARSE_DET", "0")), **part)
print(tr)
