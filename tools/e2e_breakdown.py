"""Where the end-to-end time of bench.py's e2e leg goes: create, iterations (with the F trace), state readback."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

p = gen.generate(sys.argv[1] if len(sys.argv) > 1 else "final13682")
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
hc, hp, hoc, hop, huv = map(pin, (p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv))
torch.cuda.init()
for rep in range(2):
    t0 = time.perf_counter()
    s = daba.Solver(hc, hp, hoc, hop, huv, loss=p.loss)
    t1 = time.perf_counter()
    F, _ = s.iterate(steps, F_trace=True)
    t2 = time.perf_counter()
    c, l, _ = s.state()
    t3 = time.perf_counter()
    s.close()
    t4 = time.perf_counter()
    print(f"create {t1 - t0:.3f}  iterate {t2 - t1:.3f}  state {t3 - t2:.3f}  close {t4 - t3:.3f}  "
          f"e2e {steps * p.K / (t3 - t0) / 1e9:.2f} G obs/s")
