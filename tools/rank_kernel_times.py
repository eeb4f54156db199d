"""Per-kernel times of one rank's shard at N ranks (DABA_COMM_NONE, one GPU; CUDA events around every launch),
next to the graph-replayed iteration time of the same shard."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "final13682"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
r = int(sys.argv[3]) if len(sys.argv) > 3 else 0
it = 40
p = gen.generate(cfg)
kw = dict(loss=p.loss, loss_scale=p.loss_scale, rank=r, nranks=n, comm=daba.COMM_NONE) if n > 1 else dict(loss=p.loss)
with daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, profile=1, **kw) as s:
    s.iterate(3)
    s.reset_kernel_times()
    s.iterate(it)
    kt = s.kernel_times()
    print(f"N={n} rank {r} profiled", {k: round(v[0] / it, 4) for k, v in kt.items() if v[1]},
          "sum", round(sum(v[0] for v in kt.values()) / it, 4), s.shard_info())
with daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, **kw) as g:
    g.iterate(3)
    g.objective()
    t0 = time.perf_counter()
    g.objective()
    t_obj = time.perf_counter() - t0
    t0 = time.perf_counter()
    g.iterate(it)
    g.objective()
    print(f"N={n} rank {r} graph {1e3 * (time.perf_counter() - t0 - t_obj) / it:.4f} ms/iter, launches/iter",
          g.launches_per_iteration())
