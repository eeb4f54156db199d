"""Diagnose a trajectory-parity miss: run the GPU k iterations, hand its (x^k, x^{k-1}, s, F-bar) to the oracle,
take ONE iteration on both and compare the trace row and every camera's accepted LM trial (both anchors).

    python tools/diag_trajectory.py trafalgar 0.1 34
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2305_07026_b200 as D  # noqa: E402

name, eta, k = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
p = gen.generate(name)
with D.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale, eta=eta) as s:
    s.iterate(k)
    ck, lk, _ = s.state_native(0)
    cp, lp, _ = s.state_native(1)
    sk, Fb, kk = s.schedule()
    trg = s.iterate_trace(1)
    ga, gm = s.decisions()
o = oracle.Oracle(p, eta=eta)
o.set_state(0, ck, lk)
o.set_state(1, cp, lp)
o.set_schedule(sk, Fb)
tro = o.iterate(1)
oa, om = o.decisions()
names = ["F", "Fbar", "Eacc", "restart", "Emm", "step2", "gamma", "ndeg", "noacc_acc", "noacc_mm"]
for c, nm in enumerate(names):
    g, r = trg[0, c], tro[0, c]
    print(f"{nm:10s} gpu {g:.17g} oracle {r:.17g} rel {abs(g - r) / max(abs(r), 1e-300):.3e}")
da, dm = np.nonzero(ga != oa)[0], np.nonzero(gm != om)[0]
print("acc-anchor decisions differing:", da.size, [(int(i), int(ga[i]), int(oa[i])) for i in da[:20]])
print("mm-anchor decisions differing:", dm.size, [(int(i), int(gm[i]), int(om[i])) for i in dm[:20]])
# the accelerated candidates of the differing cameras: the oracle's trial decreases around the tie
if da.size:
    ca, cm, _, _ = o.candidates(da[:5], np.zeros(0, np.int64))
    print("oracle acc candidates of the differing cameras (first rows):", ca[:2, 9:12])
