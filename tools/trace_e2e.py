"""Host-side phase breakdown of one C2 plan_step through the public API.

Runs `paraplan.Planner.plan_step` on the bench's C2 snapshot (bench.py's e2e
arm) with PARAPLAN_TRACE=2 in a child process, parses the per-step
"[paraplan] plan_step us: ..." lines the C-ABI prints (capi_internal.hpp,
PhaseClock) and prints the median time stamp of every phase, in microseconds
from the start of plan_step. Needs a GPU.

    python tools/trace_e2e.py [--steps 200]
"""
import argparse
import os
import re
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(steps: int) -> None:
    sys.path.insert(0, ROOT)
    from paper_1904_06680_b200 import import_paraplan, workloads
    pp = import_paraplan()
    w = workloads.c2(samples=1 << 20, precision=32)
    H, N = w.model.H, int(w.snapshot.field.shape[1])
    pc = pp.PlannerConfig()
    pc.H, pc.n_restarts, pc.n_candidates = H, 1, 1 << 20
    pc.precision, pc.device, pc.n_obst_pts = 32, 0, N
    planner = pp.Planner(pp.VehicleParams(), pp.MlpArchitecture([5, 2, 2]), pc)
    m = workloads.c2_mission()
    snap = pp.PlanningSnapshot()
    snap.ev_state = m.initial_state
    snap.prev_action = pp.ControlAction(0.0, pp.idle_longitudinal(pp.VehicleParams()))
    snap.goal = pp.select_goal(m, m.initial_state, 0, pp.GoalTolerance()).goal
    ev = m.initial_state
    snap.obstacle_field = pp.extrapolate(pp.sense(m, ev, w.t, N, 0.1), H, 0.1,
                                         pp.Pose2(ev.x, ev.y, ev.phi))
    for _ in range(20):
        planner.plan_step(snap, w.t)
    print("--- timed ---", file=sys.stderr, flush=True)
    wall = []
    for _ in range(steps):
        t0 = time.perf_counter()
        planner.plan_step(snap, w.t)
        wall.append((time.perf_counter() - t0) * 1e6)
    print(f"wall_us_median={statistics.median(wall):.1f}", file=sys.stderr, flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.steps)
        return
    env = dict(os.environ, PARAPLAN_TRACE="2")
    p = subprocess.run([sys.executable, __file__, "--child", "--steps", str(a.steps)],
                       env=env, capture_output=True, text=True, check=True)
    lines = p.stderr.split("--- timed ---", 1)[1].splitlines()
    phases: dict[str, list[float]] = {}
    order: list[str] = []
    for ln in lines:
        if "plan_step us:" not in ln:
            continue
        for name, us in re.findall(r"(\S+)=([0-9.]+)", ln.split("us:", 1)[1]):
            if name not in phases:
                order.append(name)
            phases.setdefault(name, []).append(float(us))
    wall = [ln for ln in lines if ln.startswith("wall_us_median=")]
    print(f"C2 plan_step, {a.steps} steps (tracing on), median phase time stamps in us:")
    prev = 0.0
    for name in order:
        t = statistics.median(phases[name])
        print(f"  {name:12s} {t:8.1f}  (+{t - prev:6.1f})")
        prev = t
    if wall:
        print("  " + wall[0])


if __name__ == "__main__":
    main()
