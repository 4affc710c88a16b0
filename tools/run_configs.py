"""Time the BASELINE.json configurations through the C-ABI (one GPU).

  C1  4096 samples, H=20, 18 static points           (single control step)
  C2  2^20 samples, H=30, 20 points (4 moving)       (bench workload)
  C3  exp4 closed loop, 2^20 samples, H=200, N=0     (per-tick latency, K ticks)
  C4  exp5_3wp lot densified to 10k points, H=200    (--c4-samples, default 2^20)
  C5  sweep points (samples x H x N)
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_06680_b200 import abi, capi, import_paraplan, workloads  # noqa: E402


def time_round(w, reps=3, refine=1):
    w.model.refine = refine
    dp = capi.DevicePlanner(w.model)
    dp.upload(w.snapshot)
    out = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        rec, _ = dp.evaluate(None, w.t, 0, 0, w.model.n_restarts, None, 0, w.model.n_candidates)
        wall = (time.perf_counter() - t0) * 1e3
        t = dp.timing()
        out.append(dict(wall_ms=wall, device_ms=t.kernel_ms, certify_ms=t.certify_ms,
                        refined=t.refined, steps=t.executed_steps, cls=int(rec[0]["cls"]),
                        fp64_rounds=t.fp64_rounds, rollout_ms=t.rollout_ms,
                        cand=int(rec[0]["candidate"])))
    best = min(out[1:], key=lambda d: d["wall_ms"])
    best["nominal_steps_per_s"] = w.samples * w.model.H / (best["wall_ms"] * 1e-3)
    # end to end through the C-ABI with host buffers: the (H+1) x N field, and
    # (C4/C5) the raw sensed points the planner extrapolates itself
    legs = [("e2e_field_ms", lambda: dp.plan_step(w.snapshot, w.t))]
    if "points" in w.extra:
        legs.append(("e2e_points_ms",
                     lambda: dp.plan_step_points(w.snapshot, w.extra["points"], w.t)))
    for name, call in legs:
        ts = []
        for _ in range(reps + 1):
            t0 = time.perf_counter()
            call()
            ts.append((time.perf_counter() - t0) * 1e3)
        best[name] = min(ts[1:])
    dp.close()
    return best


def closed_loop(samples, H, ticks, name="exp4"):
    pp = import_paraplan()
    spec = pp.builtin_scenario(name)
    c = spec.planner
    c.H, c.n_candidates, c.n_restarts = H, samples, 1
    m = spec.mission
    m.time_limit = ticks * 0.1
    t0 = time.perf_counter()
    log = pp.run_mission(m, c, spec.arch, 0)
    wall = time.perf_counter() - t0
    taus = [r.plan_time for r in log.records if r.evaluated > 0]
    return dict(ticks=len(taus), tau_avg_ms=1e3 * float(np.mean(taus)),
                tau_max_ms=1e3 * float(np.max(taus)), wall_s=wall,
                completed=bool(log.completed), tau_ms=[round(1e3 * x, 3) for x in taus])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="C1,C2,C3,C4,C5",
                    help="comma list of C1..C5, defaults (reference PlannerConfig), archs")
    ap.add_argument("--c4-samples", type=int, default=1 << 20)
    ap.add_argument("--c3-ticks", type=int, default=20)
    ap.add_argument("--fp64", type=int, default=1)
    ap.add_argument("--c5-n", default="100,1000,10000,100000")
    ap.add_argument("--c5-H", default="10,30,100")
    ap.add_argument("--c5-samples", default="12,16,20,24,26",
                    help="log2 sample counts of the C5 samples sweep (N=1000, H=30)")
    ap.add_argument("--c4-shard", type=int, default=1 << 19,
                    help="C4 per-GPU shard (2^22 samples over 8 GPUs)")
    a = ap.parse_args()
    res = {}
    which = a.which.split(",")
    if "C1" in which:
        res["C1"] = time_round(workloads.c1())
    if "C2" in which:
        res["C2"] = time_round(workloads.c2())
        if a.fp64:
            res["C2_fp64"] = time_round(workloads.c2(precision=64))
    if "defaults" in which or a.which == "C1,C2,C3,C4,C5":
        # the reference's default PlannerConfig (planner.hpp:21-35: H=200,
        # 15 restarts x 20480 candidates) on the C2 scene
        m = workloads.c2_mission()
        snap = workloads.snapshot_from_mission(m, m.initial_state, 5, 200, 20)
        w = workloads.Workload("defaults", abi.Model(H=200, n_restarts=15, n_candidates=20480),
                               snap, 5, "reference PlannerConfig defaults on the C2 scene")
        res["reference_defaults_R15x20480_H200"] = time_round(w)
    if "archs" in which:
        # C2 per network architecture (profiles/r1_archs_c2.json)
        for sizes in ((5, 2, 2), (5, 10, 2), (5, 10, 10, 2), (5, 3, 4, 2)):
            w = workloads.c2()
            w.model.layer_sizes = sizes
            r = time_round(w)
            res[str(sizes)] = {k: r[k] for k in ("wall_ms", "device_ms", "steps", "refined")}
    if "C3" in which:
        res["C3"] = closed_loop(1 << 20, 200, a.c3_ticks)
    if "C4" in which:
        res["C4"] = time_round(workloads.c4(samples=a.c4_samples), reps=1)
        # one GPU's shard of the BASELINE C4 run (2^22 samples over 8 GPUs):
        # the candidates [0, 2^19) of the 2^22-sample round
        w = workloads.c4(samples=1 << 22)
        dp = capi.DevicePlanner(w.model)
        dp.upload(w.snapshot)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            dp.evaluate(None, w.t, 0, 0, 1, None, 0, a.c4_shard)
            ts.append((time.perf_counter() - t0) * 1e3)
        tm = dp.timing()
        res["C4_shard_of_2^22_over_8"] = dict(samples=a.c4_shard, wall_ms=min(ts[1:]),
                                              device_ms=tm.kernel_ms, steps=tm.executed_steps)
        dp.close()
    if "C5" in which:
        for n_pts in map(int, a.c5_n.split(",")):
            for H in map(int, a.c5_H.split(",")):
                res[f"C5_n{n_pts}_H{H}"] = time_round(workloads.c5(1 << 20, H, n_pts), reps=1)
        for k in map(int, a.c5_samples.split(",")):
            r = time_round(workloads.c5(1 << k, 30, 1000), reps=1)
            res[f"C5_samples2^{k}_n1000_H30"] = r
    print(json.dumps(res, indent=1))
