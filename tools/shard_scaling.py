"""Per-rank device time of the DABA iteration at N ranks, measured one shard at a time on ONE GPU
(DABA_COMM_NONE: no peers, the allreduce is a local copy, the halo exchange is skipped — a measurement of the
device work each rank does, NOT of the method's iterates, and NOT including the NVLink collectives).

For N in --ranks, every rank r < N of the Final-13682-shaped problem (default partition: contiguous camera
ranges balanced by observations, plurality point owners) is created alone and timed over graph-replayed
iterations; the strong-scaling estimate is t(1) / max_r t_r(N) before communication, next to the per-rank
halo volume the NCCL exchange would move.

  python tools/shard_scaling.py [--config final13682] [--ranks 1,2,4,8] [--iters 50] [--out profiles/...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402


def time_rank(p, r, n, iters):
    kw = dict(loss=p.loss, loss_scale=p.loss_scale)
    if n > 1:
        kw.update(rank=r, nranks=n, comm=daba.COMM_NONE)
    with daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, **kw) as s:
        s.iterate(5)
        s.objective()  # synchronises
        t0 = time.perf_counter()
        s.objective()
        t_obj = time.perf_counter() - t0
        t0 = time.perf_counter()
        s.iterate(iters)
        s.objective()
        dt = time.perf_counter() - t0 - t_obj
        return 1e3 * dt / iters, s.shard_info(), s.launches_per_iteration()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="final13682")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    p = gen.generate(a.config)
    res = {"config": a.config, "K": int(p.K), "iters": a.iters, "runs": []}
    t1 = None
    for n in [int(x) for x in a.ranks.split(",")]:
        per = []
        for r in range(n):
            ms, info, lpi = time_rank(p, r, n, a.iters)
            per.append({"rank": r, "ms": ms, "cam_side_obs": info["cam_side_obs"], "pt_side_obs": info["pt_side_obs"],
                        "halo_cams": info["halo_cams"], "halo_pts": info["halo_pts"],
                        "send_bytes_per_iter": info["send_bytes_per_iter"], "launches": lpi})
            print(n, per[-1], flush=True)
        tmax = max(x["ms"] for x in per)
        if n == 1:
            t1 = tmax
        res["runs"].append({"nranks": n, "max_ms": tmax, "speedup_before_comm": t1 / tmax if t1 else None,
                            "ranks": per})
    print(json.dumps({r["nranks"]: (round(r["max_ms"], 4), round(r["speedup_before_comm"] or 0, 2))
                      for r in res["runs"]}))
    if a.out:
        with open(a.out + ".json", "w") as f:
            json.dump(res, f, indent=1)
        with open(a.out + ".md", "w") as f:
            f.write(f"# Per-rank device time at N ranks ({a.config}, one shard at a time on one B200)\n\n")
            f.write("DABA_COMM_NONE measurement mode: each rank's kernels alone, collectives excluded (the NCCL "
                    "allreduce of 96 B and the halo send/recv are not in these numbers).\n\n")
            f.write("| N | max rank ms/iter | t(1)/max t_r(N) | per-rank ms | halo send MB/iter (max) |\n"
                    "|---|---|---|---|---|\n")
            for r in res["runs"]:
                f.write(f"| {r['nranks']} | {r['max_ms']:.4f} | {r['speedup_before_comm']:.2f} | " +
                        ", ".join(f"{x['ms']:.3f}" for x in r["ranks"]) + " | " +
                        f"{max(x['send_bytes_per_iter'] for x in r['ranks']) / 1e6:.2f} |\n")


if __name__ == "__main__":
    main()
