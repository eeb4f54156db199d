"""Debug helper: n ranks as threads on one GPU through the LOCAL transport; prints each rank's failure at once."""
import faulthandler
import os
import sys
import threading
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as D  # noqa: E402

faulthandler.dump_traceback_later(90, exit=True)
name = sys.argv[1] if len(sys.argv) > 1 else "small_seq_huber"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = gen.generate(name)
key = np.random.default_rng(n).bytes(128)


def work(r):
    try:
        s = D.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale, rank=r,
                     nranks=n, comm_key=key, comm=D.COMM_LOCAL)
        print(f"rank {r} created {s.shard_info()}", flush=True)
        tr = s.iterate_trace(5)
        print(f"rank {r} F {tr[:, 0]}", flush=True)
        s.close()
    except Exception:
        print(f"rank {r} FAILED\n{traceback.format_exc()}", flush=True)


th = [threading.Thread(target=work, args=(r,)) for r in range(n)]
[t.start() for t in th]
[t.join() for t in th]
