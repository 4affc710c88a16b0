"""BASELINE.json configurations as concrete planner inputs.

Snapshots are built exactly as the reference mission loop builds them
(select_goal -> sense -> extrapolate, /root/reference/proj/src/mission.cpp:
124-144) through this repo's own host API (`paraplan._core`), then packed
into the C-ABI PODs. tests/test_workloads.py pins them bit-for-bit against
the reference's own sense/select_goal/extrapolate.

  C1  exp3_explicit without dynamic points, t=0, H=20, 4096 samples
  C2  reference sensing fixture (mission_test.cpp:54-74): 16 road-bound points
      + 4 oncoming corners at 20 km/h, t=5 -> exactly 20 points, 4 moving;
      EV 50 km/h, goal clipped to (30, 0, 0, 13.89); H=30, 2^20 samples
  C3  exp4 closed loop (forward/reverse, max steering), H=200, 2^20 samples
  C4  exp5_3wp with the lot densified to 10,000 static points, H=200, 2^22
  C5  sweep generator: samples x H x obstacle count (25% dynamic)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import abi


def _pp():
    from .python_path import import_paraplan
    return import_paraplan()


@dataclass
class Workload:
    name: str
    model: abi.Model
    snapshot: abi.Snapshot
    t: int
    description: str
    extra: dict = field(default_factory=dict)

    @property
    def samples(self) -> int:
        m = self.model
        return m.n_restarts * m.n_iter_max * m.n_candidates


def snapshot_from_mission(mission, ev, t: int, H: int, n_obst_pts: int, prev_action=None,
                          actuator_delta: float = 0.0, warm_theta=None) -> abi.Snapshot:
    """mission.cpp:124-144 through the drop-in host API."""
    pp = _pp()
    params = pp.VehicleParams()
    sel = pp.select_goal(mission, ev, 0, pp.GoalTolerance())
    pts = pp.sense(mission, ev, t, n_obst_pts, params.T_s)
    f = pp.extrapolate(pts, H, params.T_s, pp.Pose2(ev.x, ev.y, ev.phi))
    fld = np.array([[(q.x, q.y) for q in f.at(h)] for h in range(H + 1)],
                   dtype=np.float64).reshape(H + 1, f.n_points, 2)
    if prev_action is None:
        prev_action = (0.0, pp.idle_longitudinal(params))
    return abi.Snapshot(ev=(ev.x, ev.y, ev.phi, ev.v), actuator_delta=actuator_delta,
                        prev_action=prev_action,
                        goal=(sel.goal.x, sel.goal.y, sel.goal.phi, sel.goal.v), field=fld,
                        warm_theta=warm_theta)


def builtin_snapshot(name: str, t: int, H: int, n_obst_pts: int = 20,
                     drop_dynamic: bool = False) -> abi.Snapshot:
    pp = _pp()
    spec = pp.builtin_scenario(name)
    m = spec.mission
    if drop_dynamic:
        m.dynamic_points = []
    return snapshot_from_mission(m, m.initial_state, t, H, n_obst_pts)


C2_T = 5
C2_H = 30
C2_N_OBST = 20


def c2_mission_arrays():
    """C2 mission as plain arrays (no native code): waypoints (x, y, phi, v),
    static and dynamic points (x, y, heading, speed) in the world frame, EV
    state (x, y, phi, v). The reference's sensing fixture
    (mission_test.cpp:54-74)."""
    wp = np.array([[50.0, 0.0, 0.0, 50.0 / 3.6]])
    st = []
    for i in range(8):
        st.append((2.0 + 3.0 * i, -1.75, 0.0, 0.0))
        st.append((2.0 + 3.0 * i, 5.25, 0.0, 0.0))
    sp = 20.0 / 3.6
    dy = [(28.2, -1.0, math.pi, sp), (28.2, 1.0, math.pi, sp),
          (32.0, -1.0, math.pi, sp), (32.0, 1.0, math.pi, sp)]
    ev = np.array([0.0, 0.0, 0.0, 50.0 / 3.6])
    return wp, np.array(st), np.array(dy), ev


def c2_mission():
    pp = _pp()
    wp, st, dy, ev = c2_mission_arrays()
    m = pp.Mission()
    m.waypoints = [pp.GoalSetpoint(*w) for w in wp]
    m.static_points = [pp.ObstaclePoint(*q) for q in st]
    m.dynamic_points = [pp.ObstaclePoint(*q) for q in dy]
    m.initial_state = pp.VehicleState(*ev)
    return m


def c1(precision: int = abi.PP_FP32, samples: int = 4096) -> Workload:
    H = 20
    snap = builtin_snapshot("exp3_explicit", 0, H, drop_dynamic=True)
    model = abi.Model(H=H, n_restarts=1, n_candidates=samples, precision=precision)
    return Workload("C1", model, snap, 0,
                    f"exp3_explicit static road bounds ({snap.field.shape[1]} pts), t=0, H=20, "
                    f"{samples} samples")


def c2(precision: int = abi.PP_FP32, samples: int = 1 << 20) -> Workload:
    H = C2_H
    m = c2_mission()
    snap = snapshot_from_mission(m, m.initial_state, C2_T, H, C2_N_OBST)
    model = abi.Model(H=H, n_restarts=1, n_candidates=samples, precision=precision)
    return Workload("C2", model, snap, 5,
                    f"dynamic obstacle avoidance: 16 static + 4 oncoming points at 20 km/h "
                    f"(mission_test.cpp:54-74 fixture, t=5), H=30, {samples} samples")


def densified_lot(n_points: int = 10000) -> np.ndarray:
    """points spaced uniformly along the lot polylines
    (scenario.cpp:66-71)."""
    lines = [[(-6.5, -2), (-2.5, -2), (-2.5, -7), (2.5, -7), (2.5, -2), (6.5, -2)],
             [(-4, 6), (4, 6)]]
    segs = []
    for pl in lines:
        for a, b in zip(pl[:-1], pl[1:]):
            segs.append((np.array(a, float), np.array(b, float)))
    lens = np.array([np.linalg.norm(b - a) for a, b in segs])
    total = lens.sum()
    s = (np.arange(n_points) + 0.5) * total / n_points
    out = np.zeros((n_points, 4))
    cum = np.concatenate([[0.0], np.cumsum(lens)])
    for k, sk in enumerate(s):
        i = min(np.searchsorted(cum, sk, side="right") - 1, len(segs) - 1)
        a, b = segs[i]
        p = a + (b - a) * (sk - cum[i]) / lens[i]
        out[k, :2] = p
    return out


def c4(precision: int = abi.PP_FP32, samples: int = 1 << 22, n_points: int = 10000,
       H: int = 200) -> Workload:
    pp = _pp()
    spec = pp.builtin_scenario("exp5_3wp")
    m = spec.mission
    m.static_points = [pp.ObstaclePoint(*row) for row in densified_lot(n_points)]
    snap = snapshot_from_mission(m, m.initial_state, 0, H, n_points)
    ev = m.initial_state
    pts = np.array([(q.x, q.y, q.heading, q.speed) for q in
                    pp.sense(m, ev, 0, n_points, pp.VehicleParams().T_s)], dtype=np.float64)
    model = abi.Model(H=H, n_restarts=1, n_candidates=samples, n_obst_pts=n_points,
                      precision=precision)
    return Workload("C4", model, snap, 0,
                    f"reverse parking, {n_points} static lot points, H={H}, {samples} samples",
                    extra={"points": pts})


def c5(samples: int, H: int, n_points: int, precision: int = abi.PP_FP32,
       seed: int | None = None) -> Workload:
    """EV (0,0,0,50 km/h), goal (30,0,0,50 km/h); points
    uniform in xi [-10, 30], |eta| in [2.5, 10]; 25% dynamic, heading 0/pi,
    speed U(0, 15) m/s."""
    rng = np.random.default_rng(n_points if seed is None else seed)
    pts = np.zeros((n_points, 4))
    pts[:, 0] = rng.uniform(-10.0, 30.0, n_points)
    pts[:, 1] = rng.uniform(2.5, 10.0, n_points) * rng.choice([-1.0, 1.0], n_points)
    dyn = rng.random(n_points) < 0.25
    pts[dyn, 2] = rng.choice([0.0, math.pi], dyn.sum())
    pts[dyn, 3] = rng.uniform(0.0, 15.0, dyn.sum())
    snap = abi.Snapshot(ev=(0.0, 0.0, 0.0, 50.0 / 3.6), prev_action=(0.0, 0.32142857142857145),
                        goal=(30.0, 0.0, 0.0, 50.0 / 3.6), field=abi.extrapolate(pts, H))
    model = abi.Model(H=H, n_restarts=1, n_candidates=samples, n_obst_pts=n_points,
                      precision=precision)
    return Workload("C5", model, snap, 0, f"sweep point: {samples} samples, H={H}, N={n_points}",
                    extra={"points": pts})


def algorithmic_flops(layer_sizes, n_points: int, executed_steps: int, checked_states: int) -> int:
    """Algorithmic FP work of a sampling round ('Roofline'):
    per simulated step  features 9 + MLP 2*MAC + map_controls 17 + Euler 16 +
    path 6 = 48 + 2*MAC; per checked state goal box 19 + collision 6*N.
    Transcendentals (tanh per unit, tan, sincos, sqrt, wrap) are not counted."""
    s = list(layer_sizes)
    mac = sum(s[i] * s[i + 1] for i in range(len(s) - 1))
    return executed_steps * (48 + 2 * mac) + checked_states * (19 + 6 * n_points)
