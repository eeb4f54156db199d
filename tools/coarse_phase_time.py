"""NEXT-3 phase timing on Final-13682 (round-1 helper): daba_coarse_blocks, daba_coarse_solve with the stored W,
and daba_coarse_run over 1 / 2 iterations (host clock)."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import gen, paper_2305_07026_b200 as daba
from tools.coarse_common import bal_to_native, camera_sorted
p = gen.generate("final13682"); order, off = camera_sorted(p)
dev = torch.device("cuda:0")
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)
oc, op, uv, offt = t(np.asarray(p.obs_cam)[order], torch.int32), t(np.asarray(p.obs_pt)[order], torch.int32), t(np.asarray(p.obs_uv).reshape(-1,2)[order], torch.float64), t(off, torch.int64)
c0, l0 = t(bal_to_native(p.cams), torch.float64), t(np.asarray(p.pts).reshape(-1,3), torch.float64)
def tm(f, n=3):
    f(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return 1e3*(time.perf_counter()-t0)/n
b = daba.coarse_blocks(c0, l0, op, uv, offt, loss=p.loss)
print("blocks ms", tm(lambda: daba.coarse_blocks(c0, l0, op, uv, offt, loss=p.loss)))
print("solve ms (W stored, 30 it)", tm(lambda: daba.coarse_solve(b, oc, op, offt, max_iter=30, tol=1e-4)))
print("solve info", daba.coarse_solve(b, oc, op, offt, max_iter=30, tol=1e-4)[2])
for n in (1, 2, 1):
    c, l = c0.clone(), l0.clone(); torch.cuda.synchronize(); t0=time.perf_counter()
    daba.coarse_run(c, l, oc, op, uv, offt, n, loss=p.loss, pcg_max_iter=30, pcg_tol=1e-4); torch.cuda.synchronize()
    print("run", n, "ms", 1e3*(time.perf_counter()-t0))
