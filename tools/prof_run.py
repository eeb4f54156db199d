"""Minimal DABA run for ncu: generate a config, create one context, run warm-up + N iterations."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="final13682")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--shuffle", action="store_true")
a = ap.parse_args()
p = gen.generate(a.config, shuffle_points=a.shuffle)
s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, use_graph=0)
s.iterate(a.iters)
print("F", s.objective())
s.close()
