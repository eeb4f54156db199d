#!/usr/bin/env python
"""DABA hot-path benchmark (BASELINE.json metric: observations/sec per DABA iteration, % HBM roofline).

One step = one DABA iteration (Algorithm 1) over the whole synthetic BAL Final-13682-shaped problem
(BASELINE.json configs[3]: 13,682 cameras, 4,456,117 points, 28,987,644 observations, Huber loss), fp64.
N = 1: one B200.  N > 1 (torchrun, one rank per GPU): the same problem partitioned across the ranks (strong
scaling; NCCL halo exchange + one allreduce per iteration).  --config weak_slab (configs[4], Cauchy): N slabs of
31.25M observations at N GPUs (weak scaling).  --restart device: the paper's decentralized per-device restart
(reading DN1) instead of the global test.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config final13682] [--restart global|device]
                  [--impl reference]

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "observations/sec per DABA iteration"
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP64 peak: DFMA/s measured on this pool's B200 (tools/dmma_micro.cu, independent chains, 148 SMs:
# profiles/r02_fp64_micro.log, 17.71 T DFMA/s; DMMA m8n8k4 18.4 T FMA/s — no faster) -> FLOP/s = 2 x DFMA/s
FP64_FLOPS_PEAK = 2 * 17.71e12

# Algorithmic work, per iteration at K observations, N points, M cameras:
#   bytes: K * 20 (u 16 B + point index 4 B) + N * 96 (read l^k and l^{k-1}, write l_acc and l_mm; 24 B each)
#          + M * 500 (camera copies and moments)
#   k_cam_pass's own share: K * 20 + N * 48 (reads the two anchors' points once) + M * 256 (the two anchor cameras)
#   FP64: 150.5 FLOP per observation and anchor in k_cam_pass — ncu SASS opcode counts of one launch on
#   Final-13682 (DFMA 57.58 x 2 + DMUL 24.74 + DADD 10.59 thread instructions per observation and anchor;
#   profiles/r02_cam_pass_sass_counts.txt), i.e. 301.0 FLOP per observation and iteration.
ALG_BYTES_ITER = lambda K, N, M: 20 * K + 96 * N + 500 * M
ALG_BYTES = {"k_cam_pass": lambda K, N, M: 20 * K + 48 * N + 256 * M}
FLOP_PER_ANCHOR_OBS = 150.5
TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="final13682", help="a gen config name or the path of a BAL file")
    ap.add_argument("--restart", default="global", choices=["global", "device"])
    # test plumbing: "none" runs every rank's shard alone (DABA_COMM_NONE: no collectives, NOT the method's
    # iterates) so that the multi-rank driver logic can be exercised on a one-GPU box
    ap.add_argument("--comm", default="nccl", choices=["nccl", "none"])
    ap.add_argument("--impl", default="daba", choices=["daba", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p:
            self.p.terminate()
            out, _ = self.p.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def peaks():
    try:
        with open(MEASURED) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


WEAK = {"weak_slab"}  # BASELINE.json configs[4]: per-GPU slab fixed, N slabs at N GPUs (weak scaling)


def make_problem(config, world):
    import gen
    if os.path.isfile(config):  # a BAL file (the paper's datasets, when present): read natively, Huber loss
        import paper_2305_07026_b200 as daba
        b = daba.read_bal(config)
        cams, uv = daba.bal_to_paper(b.cams, b.obs_uv)
        return gen.Problem(os.path.basename(config), cams, b.pts, b.obs_cam, b.obs_pt, uv, cams, b.pts,
                           daba.LOSS_HUBER, 1.0), "strong"
    if config in WEAK:
        cM, cN, cK = gen.CONFIGS[config][:3]
        return gen.generate(config, M=cM * world, N=cN * world, K=cK * world), "weak"
    return gen.generate(config), "strong"


def sample_problem(p, max_obs):
    """Induced sub-problem on the first cameras whose observations total <= max_obs (for the CPU oracle)."""
    import numpy as np

    import gen
    counts = np.bincount(p.obs_cam, minlength=p.M)
    m = int(np.searchsorted(np.cumsum(counts), max_obs))
    m = max(1, min(m, p.M))
    sel = p.obs_cam < m
    pts_used = np.unique(p.obs_pt[sel])
    remap = np.full(p.N, -1, np.int64)
    remap[pts_used] = np.arange(pts_used.size)
    return gen.Problem(p.name + f"[cams<{m}]", p.cams[:m].copy(), p.pts[pts_used].copy(),
                       p.obs_cam[sel].astype(np.int32), remap[p.obs_pt[sel]].astype(np.int32), p.obs_uv[sel].copy(),
                       p.gt_cams[:m].copy(), p.gt_pts[pts_used].copy(), p.loss, p.loss_scale)


def run_oracle_sample(p, max_obs, iters):
    import oracle
    sp = sample_problem(p, max_obs)
    o = oracle.Oracle(sp)
    t0 = time.perf_counter()
    o.iterate(iters)
    dt = time.perf_counter() - t0
    o.close()
    return sp, dt


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import numpy as np

    import gen

    if a.impl == "reference":
        # The reference arm is the CPU oracle, as it stands, on the box's host cores (rank 0 only).
        if rank != 0:
            return
        p, _ = make_problem(a.config, 1)
        sp = sample_problem(p, 60_000)
        import oracle
        o = oracle.Oracle(sp)
        o.iterate(max(a.warmup, 0))
        t0 = time.perf_counter()
        o.iterate(a.steps)
        dt = time.perf_counter() - t0
        v = a.steps * sp.K / dt
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "obs/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": ("bal file" if os.path.isfile(a.config) else "synthetic"),
            "config": {"workload": a.config, "sample": sp.name, "sample_obs": int(sp.K)},
            "cpu_baseline": {"value": v, "unit": "obs/s", "cores": 1, "kind": "oracle",
                             "sample": f"{sp.name}: {sp.K} observations, {a.steps} iterations"},
            "e2e": {"value": v, "unit": "obs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist

    import paper_2305_07026_b200 as daba

    local = local % max(torch.cuda.device_count(), 1) if a.comm == "none" else local
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    p, scaling = make_problem(a.config, world)

    def fresh_key():
        # every context gets its own NCCL communicator, hence its own unique id (rank 0 draws, all receive)
        if world == 1 or a.comm == "none":
            return None
        obj = [daba.comm_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    stream = torch.cuda.Stream(device=local)
    kw = dict(loss=p.loss, loss_scale=p.loss_scale, rank=rank, nranks=world, device=local,
              comm=daba.COMM_NONE if a.comm == "none" else daba.COMM_NCCL,
              restart_scope=1 if a.restart == "device" else 0)

    # ---------------- device-resident timed region (production path: one CUDA graph per iteration)
    s = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, stream=stream.cuda_stream, comm_key=fresh_key(),
                    **kw)
    lpi = s.launches_per_iteration()
    # three repeats of the K timed steps (the median is reported); each repeat is bracketed by
    # a barrier and a synchronize, and its time is the max over ranks
    reps = []
    with torch.cuda.stream(stream):
        s.iterate(a.warmup)
        torch.cuda.synchronize()
        with Clocks(local) as clk:
            time.sleep(0.3)
            for _ in range(3):
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                s.iterate(a.steps)
                e1.record(stream)
                torch.cuda.synchronize()
                r_ms = e0.elapsed_time(e1)
                if world > 1:
                    t = torch.tensor([r_ms], dtype=torch.float64)
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    r_ms = float(t.item())
                reps.append(r_ms)
        if world > 1:
            dist.barrier()
    ms = statistics.median(reps)
    F_end = s.objective()
    info = s.shard_info()
    s.close()

    # ---------------- per-kernel times: the same steps with CUDA events around every launch (same stream)
    sp_ = daba.Solver(p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv, stream=stream.cuda_stream, profile=1,
                      comm_key=fresh_key(), **kw)
    with torch.cuda.stream(stream):
        sp_.iterate(a.warmup)
        torch.cuda.synchronize()
        sp_.reset_kernel_times()
        if world > 1:
            dist.barrier()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        sp_.iterate(a.steps)
        q1.record(stream)
        torch.cuda.synchronize()
    prof_ms = q0.elapsed_time(q1)
    kt = sp_.kernel_times()
    sp_.close()

    # ---------------- e2e through the public API from pinned host buffers
    e2e = None
    if not a.no_e2e:
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
        hc, hpnt, hoc, hop, huv = map(pin, (p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv))
        key = fresh_key()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        se = daba.Solver(hc, hpnt, hoc, hop, huv, stream=stream.cuda_stream, comm_key=key, **kw)
        t_c = time.perf_counter()
        Ftr, _ = se.iterate(a.steps, F_trace=True)
        t_i = time.perf_counter()
        cams_out, pts_out, _ = se.state()
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        phases = {"create_s": round(t_c - t0, 4), "iterate_s": round(t_i - t_c, 4), "state_s": round(te - (t_i - t0), 4)}
        se.close()
        if world > 1:
            t = torch.tensor([te], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        h2d = (hc.nbytes + hpnt.nbytes + hoc.nbytes + hop.nbytes + huv.nbytes) / a.steps
        d2h = (8 * a.steps + 1 * a.steps + cams_out.nbytes + pts_out.nbytes) / a.steps
        e2e = {"value": a.steps * p.K / te, "unit": "obs/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "includes": "daba_create (host shard plan + H2D) + iterations with "
               "per-step F readback + daba_get_state", "phases": phases}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---------------- cpu baseline: the oracle on a bounded sample, rank 0, N = 1 only
    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        spb, dt = run_oracle_sample(p, 2_000_000, 2)
        cpu = {"value": 2 * spb.K / dt, "unit": "obs/s", "cores": 1, "kind": "oracle",
               "sample": f"{spb.name}: {spb.K} of {p.K} observations, 2 iterations, single thread",
               "host_cores": os.cpu_count(), "cpu_model": cpu_model()}

    value = a.steps * p.K / (ms * 1e-3)
    hbm, hbm_src = peaks()
    K_c, K_p = info["cam_side_obs"], info["pt_side_obs"]
    N_l, M_l = info["own_pts"] + info["halo_pts"], info["own_cams"]
    kt = {k: v for k, v in kt.items() if v[1] > 0}
    kshare = {k: round(v[0] / prof_ms, 4) for k, v in kt.items()}
    # dominant kernel: k_cam_pass (FP64-bound), timed live with events on the library's stream
    dname = "k_cam_pass" if "k_cam_pass" in kt else max(kt.items(), key=lambda kv: kv[1][0])[0]
    dms, dl = kt[dname]
    per_launch_ms = dms / max(dl, 1)
    traffic, fp64_pipe = None, None
    try:  # (captured on the single-GPU Final-13682 workload: it applies only to that launch)
        if world == 1 and a.config == "final13682":
            tj = json.load(open(TRAFFIC)).get(dname, {})
            traffic, fp64_pipe = tj.get("dram_bytes_per_launch"), tj.get("fp64_pipe_pct")
    except Exception:
        pass
    roof = None
    if dname == "k_cam_pass":
        flop = FLOP_PER_ANCHOR_OBS * 2 * K_c
        ach = flop / (per_launch_ms * 1e-3) / 1e12
        kb = ALG_BYTES["k_cam_pass"](K_c, N_l, M_l)
        it_b = ALG_BYTES_ITER(K_c, N_l, M_l)
        it_s = ms / a.steps * 1e-3
        roof = {"bound": "alu", "achieved": round(ach, 3), "peak": round(FP64_FLOPS_PEAK / 1e12, 2), "unit": "TFLOP/s",
                "frac": round(ach * 1e12 / FP64_FLOPS_PEAK, 4), "traffic": traffic, "kernel": dname,
                "flop_per_launch": int(flop), "kernel_ms_per_launch": round(per_launch_ms, 5),
                "peak_source": "measured FP64 DFMA peak (tools/dmma_micro.cu, profiles/r02_fp64_micro.log)",
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, one launch)" if traffic else None,
                "fp64_pipe_pct_ncu": fp64_pipe,
                "hbm_algorithmic": {"bytes_per_launch": int(kb), "achieved_gbs": round(kb / (per_launch_ms * 1e-3) / 1e9, 1),
                                    "peak_gbs": hbm, "frac": round(kb / (per_launch_ms * 1e-3) / 1e9 / hbm, 4),
                                    "peak_source": hbm_src},
                "iteration": {"bytes": int(it_b), "achieved_gbs": round(it_b / it_s / 1e9, 1),
                              "hbm_frac": round(it_b / it_s / 1e9 / hbm, 4),
                              "flop": int(FLOP_PER_ANCHOR_OBS * 2 * K_c),
                              "fp64_frac": round(FLOP_PER_ANCHOR_OBS * 2 * K_c / it_s / FP64_FLOPS_PEAK, 4)}}
    out = {
        "metric": METRIC, "value": value, "unit": "obs/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms / a.steps, "iterations_per_s": a.steps / (ms * 1e-3),
        "repeats_ms_per_step": [round(r / a.steps, 5) for r in reps], "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": ("bal file" if os.path.isfile(a.config) else "synthetic"),
        "config": {"workload": a.config if scaling == "strong" else f"{a.config} x{world}", "cameras": p.M, "points": p.N, "observations": int(p.K),
                   "loss": ["trivial", "huber", "cauchy"][p.loss], "parallelism": f"camera-partitioned x{world}",
                   "restart": a.restart,
                   "l2": (f"inputs larger than L2 (observation streams {20 * p.K / 1e9:.2f} GB, point states "
                          f"4 x {32 * p.N / 1e6:.0f} MB)") if 20 * p.K > 126e6 else
                         "small config: inputs fit in L2 (not a benchmark workload)",
                   "F_end": F_end},
        "roofline": roof,
        "kernel_share": kshare,
        "profiled_ms_per_step": prof_ms / a.steps,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": lpi * a.steps,
        "clocks": clk.summary(),
        "shard": info,
    }
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
