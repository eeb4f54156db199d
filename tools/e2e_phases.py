"""daba_create / iterate / get_state phases from pinned host buffers (the bench's e2e path) with DABA_TIMING's
per-phase breakdown of daba_create on stderr."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "final13682"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = gen.generate(cfg)
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
hc, hp, hoc, hop, huv = map(pin, (p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = daba.Solver(hc, hp, hoc, hop, huv, loss=p.loss)
    t1 = time.perf_counter()
    F, _ = s.iterate(steps, F_trace=True)
    t2 = time.perf_counter()
    c, l, _ = s.state()
    t3 = time.perf_counter()
    s.close()
    print(f"rep {rep}: create {t1 - t0:.4f} s, {steps} iterations {t2 - t1:.4f} s, state {t3 - t2:.4f} s, "
          f"e2e {steps * p.K / (t3 - t0) / 1e9:.2f} G obs/s", flush=True)
