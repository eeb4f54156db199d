"""Iterations-to-F_Delta harness and performance profiles (§7.2 "Efficiency", eq. Fdelta P:L600-606,
Fig. 3) on synthetic problem suites, through the C-ABI.

Methods: DABA with the global restart test (D2), DABA with the decentralized per-device restart over R ranks
(reading DN1; R ranks as host threads on one GPU, LOCAL transport), and DUBA, the ablation without acceleration
or restart (x^{k+1} always from eq. update_mm).  F_ref is the smallest objective of a long DABA run
(--ref-iters; the paper takes F_ref from Ceres, which is out of scope here), and F_Delta(p) = F_ref +
Delta (F_init - F_ref) with Delta = 1e-4 as in the paper's performance profiles.

  python tools/perf_profile.py [--iters 1500] [--ranks 4] [--out profiles/r01_perf_profile]
"""
import argparse
import json
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

SUITE = [("small_huber", 0), ("small_huber", 1), ("small_cauchy", 0), ("small_cauchy", 1), ("small_seq_huber", 0),
         ("small_seq_huber", 1), ("tiny_seq", 0), ("ladybug49", 0), ("trafalgar_1m", 0), ("venice1778_1m", 0)]


def run_single(p, iters, **kw):
    with daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale, **kw) as s:
        return s.iterate_trace(iters)[:, daba.daba.TR_F]


def run_ranks(p, iters, ranks):
    key = np.random.default_rng(ranks).bytes(128)
    out, err = [None] * ranks, []

    def work(r):
        try:
            with daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, loss=p.loss, loss_scale=p.loss_scale,
                             rank=r, nranks=ranks, comm_key=key, comm=daba.COMM_LOCAL,
                             restart_scope=daba.RESTART_DEVICE) as s:
                out[r] = s.iterate_trace(iters)[:, daba.daba.TR_F]
        except Exception as e:  # pragma: no cover
            err.append(e)
    th = [threading.Thread(target=work, args=(r,)) for r in range(ranks)]
    [t.start() for t in th]
    [t.join() for t in th]
    if err:
        raise err[0]
    return out[0]


def first_below(F, target):
    idx = np.nonzero(F <= target)[0]
    return int(idx[0]) if idx.size else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=1500)
    ap.add_argument("--ranks", type=int, default=4)
    ap.add_argument("--delta", default="1e-2,1e-3,1e-4")
    ap.add_argument("--ref-iters", type=int, default=15000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    methods = {"DABA": lambda p: run_single(p, a.iters),
               f"DABA per-device x{a.ranks}": lambda p: run_ranks(p, a.iters, a.ranks),
               "DUBA": lambda p: run_single(p, a.iters, accelerate=0)}
    deltas = [float(x) for x in a.delta.split(",")]
    rows = []
    for name, seed in SUITE:
        p = gen.generate(name, seed=None if seed == 0 else 0x5EED + seed)
        traces = {m: f(p) for m, f in methods.items()}
        F_init = float(next(iter(traces.values()))[0])
        F_ref = float(min(min(t.min() for t in traces.values()), run_single(p, a.ref_iters).min()))
        its = {}
        for d in deltas:
            target = F_ref + d * (F_init - F_ref)  # eq. Fdelta
            its[str(d)] = {m: first_below(t, target) for m, t in traces.items()}
        rows.append({"problem": f"{name}#{seed}", "M": p.M, "N": p.N, "K": int(p.K), "F_init": F_init,
                     "F_ref": F_ref, "iters_to_F_delta": its, "F_final": {m: float(t[-1]) for m, t in traces.items()}})
        print(rows[-1]["problem"], its, flush=True)
    grid = [10, 25, 50, 100, 200, 400, 800, 1600, a.iters]
    profile = {str(d): {m: [sum(1 for r in rows if r["iters_to_F_delta"][str(d)][m] is not None
                                and r["iters_to_F_delta"][str(d)][m] <= k) / len(rows) for k in grid]
                        for m in methods} for d in deltas}
    res = {"deltas": deltas, "iters": a.iters, "grid": grid, "profile": profile, "problems": rows,
           "F_ref": f"smallest F of a {a.ref_iters}-iteration DABA run (or of any method)"}
    print(json.dumps(profile))
    if a.out:
        with open(a.out + ".json", "w") as f:
            json.dump(res, f, indent=1)
        with open(a.out + ".md", "w") as f:
            f.write("# Iterations to F_Delta and performance profiles (eq. Fdelta P:L600-606, Fig. 3)\n\n")
            f.write("F_ref = smallest F of a %d-iteration DABA run; budget %d iterations; synthetic suite; one B200; "
                    "per-device DABA runs its ranks as threads on the same GPU.  — = not reached.\n" %
                    (a.ref_iters, a.iters))
            for d in deltas:
                f.write(f"\n## Delta = {d:g}\n\n| problem | K | " + " | ".join(methods) + " |\n|---|---|" +
                        "---|" * len(methods) + "\n")
                for r in rows:
                    v = r["iters_to_F_delta"][str(d)]
                    f.write(f"| {r['problem']} | {r['K']} | " +
                            " | ".join(str(v[m]) if v[m] is not None else "—" for m in methods) + " |\n")
                f.write("\nFraction of problems solved by iteration k:\n\n| k | " + " | ".join(methods) +
                        " |\n|---|" + "---|" * len(methods) + "\n")
                for q, k in enumerate(grid):
                    f.write(f"| {k} | " + " | ".join(f"{profile[str(d)][m][q]:.2f}" for m in methods) + " |\n")


if __name__ == "__main__":
    main()
