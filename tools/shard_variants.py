"""A/B of create-time knobs on the per-rank device time at N ranks (one shard at a time on one GPU, DABA_COMM_NONE;
see tools/shard_scaling.py).  Each variant is a set of DABA_* environment knobs read by daba_create.

    python tools/shard_variants.py [--config final13682] [--ranks 1,8] [--iters 40] "DABA_CHUNK_ORDER=1" ...
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from tools.shard_scaling import time_rank  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="final13682")
ap.add_argument("--ranks", default="1,8")
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("variants", nargs="*", default=[""])
a = ap.parse_args()
p = gen.generate(a.config)
base_env = dict(os.environ)
for v in a.variants:
    os.environ.clear()
    os.environ.update(base_env)
    for kv in v.split():
        k, x = kv.split("=")
        os.environ[k] = x
    row = {"variant": v or "default"}
    for n in [int(x) for x in a.ranks.split(",")]:
        ts = [time_rank(p, r, n, a.iters)[0] for r in range(n)]
        row[f"N{n}_max_ms"] = round(max(ts), 4)
        row[f"N{n}_ranks"] = [round(t, 4) for t in ts]
    if "N1_max_ms" in row:
        for n in [int(x) for x in a.ranks.split(",") if x != "1"]:
            row[f"N{n}_speedup"] = round(row["N1_max_ms"] / row[f"N{n}_max_ms"], 3)
    print(json.dumps(row), flush=True)
