"""A short DABA run for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): one context on a small
config, a few graph-free iterations (so every kernel launch is visible to the tool), the state read back, plus the
multi-rank LOCAL path (2 ranks as threads) that exercises k_pt_boundary, k_unpack and the halo buffers."""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ladybug49"
p = gen.generate(name)
with D.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, use_graph=0) as s:
    tr = s.iterate_trace(4)
    s.state()
    s.pixel_error()
print("one rank F", tr[:, 0])
with D.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss) as s:  # graph path
    s.iterate(3)
key = np.random.default_rng(2).bytes(128)
out = {}


def work(r):
    with D.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, rank=r, nranks=2, comm_key=key,
                  comm=D.COMM_LOCAL, use_graph=0) as s:
        out[r] = s.iterate_trace(3)[:, 0]


th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
print("two ranks F", out)
