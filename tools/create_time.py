"""Host-side cost of daba_create on a config: shard planning alone (daba_plan_create) and the whole create."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "final13682"
p = gen.generate(cfg)
t0 = time.perf_counter()
pl = daba.Plan(p.M, p.N, p.obs_cam, p.obs_pt)
t1 = time.perf_counter()
del pl
for rep in range(2):
    t2 = time.perf_counter()
    s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss)
    t3 = time.perf_counter()
    s.iterate(1)
    s.objective()
    t4 = time.perf_counter()
    s.close()
    print(f"{cfg}: plan {t1 - t0:.3f} s, create {t3 - t2:.3f} s, first iteration (graph capture) {t4 - t3:.3f} s")
