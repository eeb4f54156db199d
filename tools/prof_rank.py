"""One rank's shard of a config at N ranks, alone on one GPU (DABA_COMM_NONE measurement mode), for ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="final13682")
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--nranks", type=int, default=8)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
p = gen.generate(a.config)
s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, rank=a.rank, nranks=a.nranks,
                comm=daba.COMM_NONE, use_graph=0)
s.iterate(a.iters)
print("F", s.objective(), s.shard_info())
s.close()
