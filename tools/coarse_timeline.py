"""GPU timeline of a short NEXT-3 run (torch.profiler / CUPTI): kernel and copy time versus wall time per coarse
iteration, and the largest idle gaps — where the host-driven loop leaves the GPU waiting."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402
from tools.coarse_common import bal_to_native, camera_sorted  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "final13682"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = gen.generate(cfg)
order, off = camera_sorted(p)
dev = torch.device("cuda:0")
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
args = (t(np.asarray(p.obs_cam)[order], torch.int32), t(np.asarray(p.obs_pt)[order], torch.int32),
        t(np.asarray(p.obs_uv).reshape(-1, 2)[order], torch.float64), t(off, torch.int64))
c0, l0 = t(bal_to_native(p.cams), torch.float64), t(np.asarray(p.pts).reshape(-1, 3), torch.float64)
kw = dict(loss=p.loss, scale=p.loss_scale, pcg_max_iter=3, pcg_tol=1e-1, mm_always=0, keep_scratch=1)
daba.coarse_run_part(c0.clone(), l0.clone(), *args, 1, **kw)
cams, pts = c0.clone(), l0.clone()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    daba.coarse_run_part(cams, pts, *args, iters, **kw)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
busy, last_end, gaps = 0.0, None, []
cur_s, cur_e = None, None
for s, e, n in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, n))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0
by = {}
for s, e, n in iv:
    k = n.replace("(anonymous namespace)::", "").split("(")[0][:60]
    by[k] = by.get(k, 0) + (e - s)
print(f"wall {1e3 * wall / iters:.3f} ms/iter, GPU span {span / 1e3 / iters:.3f} ms/iter, busy {busy / 1e3 / iters:.3f} "
      f"ms/iter, idle {(span - busy) / 1e3 / iters:.3f} ms/iter in {len(gaps)} gaps")
gaps.sort(reverse=True)
print("largest gaps (us, next op):", [(round(g, 1), n[:40]) for g, n in gaps[:12]])
print("gap histogram (us):", np.histogram([g for g, _ in gaps], bins=[0, 5, 10, 20, 50, 100, 1000, 1e6])[0].tolist())
for k, v in sorted(by.items(), key=lambda x: -x[1])[:16]:
    print(f"  {k:50s} {v / 1e3 / iters:8.3f} ms/iter")
