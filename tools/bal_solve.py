"""Solve a BAL dataset with DABA on the GPU and report the paper's accuracy metric (Table 2
P:L536-545: mean reprojection error in pixels, initial and after the iterations).

  python tools/bal_solve.py problem.txt [--iters 1000] [--loss huber --scale 1] [--out solved.txt]
  python tools/bal_solve.py --synthetic [--iters 300]     # writes a synthetic distorted BAL scene first

Pipeline (all product code): daba_bal_read (native parser) -> daba_bal_to_paper (convention map, Q15)
-> daba_create / daba_iterate -> daba_pixel_error (GPU) -> daba_get_state -> daba_paper_to_bal -> daba_bal_write.
"""
import argparse
import json
import os
import sys
import tempfile
import time



sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_07026_b200 as D  # noqa: E402

LOSSES = {"trivial": D.LOSS_TRIVIAL, "huber": D.LOSS_HUBER, "cauchy": D.LOSS_CAUCHY}


def synthetic(path, seed=None):
    """The generator's Ladybug-49-shaped problem (perturbed initial state, pixel noise, outliers) as a BAL file."""
    import gen
    p = gen.generate("ladybug49", seed=seed)
    cams, uv = D.paper_to_bal(p.cams, p.obs_uv)
    D.write_bal(path, D.BalProblem(cams, p.pts, p.obs_cam, p.obs_pt, uv))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path", nargs="?")
    ap.add_argument("--synthetic", action="store_true")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--loss", default="trivial", choices=list(LOSSES))
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--report-every", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    path = a.path
    if a.synthetic:
        path = os.path.join(tempfile.mkdtemp(), "synthetic_bal.txt")
        synthetic(path)
    if not path:
        ap.error("a BAL file or --synthetic")
    t0 = time.perf_counter()
    b = D.read_bal(path)
    t_read = time.perf_counter() - t0
    cams, uv = D.bal_to_paper(b.cams, b.obs_uv)
    rows = []
    with D.Solver(cams, b.pts, b.obs_cam, b.obs_pt, uv, loss=LOSSES[a.loss], loss_scale=a.scale) as s:
        e0 = s.pixel_error()
        rows.append({"iter": 0, "mean_px": e0["mean"], "F": s.objective()})
        step = a.report_every or a.iters
        t1 = time.perf_counter()
        done = 0
        while done < a.iters:
            n = min(step, a.iters - done)
            s.iterate(n)
            done += n
            e = s.pixel_error()
            rows.append({"iter": done, "mean_px": e["mean"], "F": s.objective()})
        t_iter = time.perf_counter() - t1
        c_out, p_out, _ = s.state()
    res = {"file": path, "M": b.M, "N": b.N, "K": b.K, "read_s": round(t_read, 3), "iterate_s": round(t_iter, 3),
           "init_mean_px": e0["mean"], "final_mean_px": rows[-1]["mean_px"], "behind_camera": e0["behind"],
           "trace": rows}
    if a.out:
        cb, ub = D.paper_to_bal(c_out, uv)
        D.write_bal(a.out, D.BalProblem(cb, p_out, b.obs_cam, b.obs_pt, ub))
        res["out"] = a.out
    print(json.dumps(res))


if __name__ == "__main__":
    main()
