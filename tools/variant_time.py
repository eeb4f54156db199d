"""Time the iteration kernels of the current libdaba.so (or $DABA_LIB) on a config: per-kernel ms per iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "final13682"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = gen.generate(cfg)
s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, profile=1)
s.iterate(3)
s.reset_kernel_times()
s.iterate(n)
kt = s.kernel_times()
tot = sum(v[0] for v in kt.values()) / n
print(os.environ.get("DABA_LIB", "default"), f"total {tot:.4f} ms/iter", {k: round(v[0] / n, 4) for k, v in kt.items()})
s.close()
# graph-replayed iterations (production path), wall clock around n iterations minus one objective evaluation
import time  # noqa: E402
g = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss)
g.iterate(3)
g.objective()
t0 = time.perf_counter()
g.objective()
t_obj = time.perf_counter() - t0
t0 = time.perf_counter()
g.iterate(n)
g.objective()
dt = time.perf_counter() - t0 - t_obj
print(os.environ.get("DABA_LIB", "default"), f"graph {1e3 * dt / n:.4f} ms/iter")
