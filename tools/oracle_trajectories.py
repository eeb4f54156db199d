"""Write 50-iteration oracle trajectories of the full-size configs into tests/golden/ (CPU only).

TEST INFRASTRUCTURE: this script calls only gen/ (seeded inputs) and oracle/ (the CPU checker); nothing here
comes from the CUDA path.  For each (config, eta) it runs Algorithm 1 for 50 iterations
in the single-threaded oracle and stores
  - the whole trace (F, F-bar, E_acc, restart, E_mm, ... per iteration; oracle.TR_* columns),
  - x^50 of a seeded sample of cameras (native 15 doubles) and points (3 doubles),
so that tests/test_gpu_trajectories.py can hold the GPU's free-running trajectory to the north star's bar
(F within 1e-10 relative every iteration, states within 1e-8 after 50 iterations) at sizes where running the
oracle beside the GPU test would take an hour.

    python tools/oracle_trajectories.py [config ...] [--eta 0.1 1.0] [--jobs 8]
"""
from __future__ import annotations

import argparse
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = ["trafalgar_1m", "venice1778_1m", "trafalgar", "venice1778", "final13682", "weak_slab"]
ITERS = 50
N_CAM_SAMPLE = 2000
N_PT_SAMPLE = 20000
SAMPLE_SEED = 0x2305


def golden_path(name: str, eta: float) -> str:
    return os.path.join(ROOT, "tests", "golden", f"traj_{name}_eta{eta:g}.npz")


def sample_ids(n: int, k: int, salt: int) -> np.ndarray:
    if n <= k:
        return np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(SAMPLE_SEED + salt)
    return np.sort(rng.choice(n, size=k, replace=False)).astype(np.int64)


def run(job):
    name, eta = job
    import gen
    import oracle

    t0 = time.time()
    p = gen.generate(name)
    o = oracle.Oracle(p, eta=eta)
    F0 = o.objective()
    tr = o.iterate(ITERS)
    cams, pts = o.state(0)
    ci = sample_ids(p.M, N_CAM_SAMPLE, 1)
    pi = sample_ids(p.N, N_PT_SAMPLE, 2)
    np.savez_compressed(golden_path(name, eta), config=name, eta=eta, iterations=ITERS, M=p.M, N=p.N, K=p.K,
                        F0=F0, trace=tr, cam_ids=ci, cams=cams[ci], pt_ids=pi, pts=pts[pi],
                        source="tools/oracle_trajectories.py (oracle/ only)")
    o.close()
    return f"{name} eta={eta:g}: {time.time() - t0:.0f} s, F {tr[0, 0]:.6e} -> {tr[-1, 0]:.6e}, " \
           f"restarts {int(tr[:, oracle.TR_RESTART].sum())}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=CONFIGS)
    ap.add_argument("--eta", nargs="*", type=float, default=[0.1, 1.0])
    ap.add_argument("--jobs", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    jobs = [(c, e) for c in a.configs for e in a.eta]
    # longest first so that the pool finishes together
    order = {c: i for i, c in enumerate(CONFIGS)}
    jobs.sort(key=lambda j: -order.get(j[0], 0))
    with mp.Pool(min(a.jobs, len(jobs))) as pool:
        for line in pool.imap_unordered(run, jobs):
            print(line, flush=True)


if __name__ == "__main__":
    main()
