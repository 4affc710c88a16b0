"""Drop-in proof on the device: the reference's planner tests
(/root/reference/proj/tests/planner_test.cpp), its Python smoke test
(tests/python/test_smoke.py) and its self-checks, restated against this
repo's `paraplan` module, whose Planner.plan_step runs the sm_100a kernel."""
from __future__ import annotations

import math
import random

import numpy as np
import pytest

from oracle.oracle import Ref
from paper_1904_06680_b200 import abi

pytestmark = pytest.mark.gpu
PI = math.pi


def snapshot_towards(pp, goal, v0, H):  # planner_test.cpp:14-21
    s = pp.PlanningSnapshot()
    s.ev_state = pp.VehicleState(0.0, 0.0, 0.0, v0)
    s.prev_action = pp.ControlAction(0.0, 0.0)
    s.goal = pp.GoalSetpoint(*goal)
    s.obstacle_field = pp.extrapolate([], H, 0.1, pp.Pose2(0, 0, 0))
    return s


def cfg(pp, **kw):
    c = pp.PlannerConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def planner(pp, **kw):
    return pp.Planner(pp.VehicleParams(), pp.MlpArchitecture([5, 2, 2]), cfg(pp, **kw))


def test_goal_satisfied_at_start(pp):
    p = planner(pp, H=40)
    s = snapshot_towards(pp, (0, 0, 0, 0), 0.0, 40)
    rnd = random.Random(31)
    for _ in range(20):
        r = p.rollout([rnd.uniform(-3, 3) for _ in range(18)], s)
        assert r.reached and r.t_goal == 0 and not r.collided and len(r.trajectory) == 1


def test_obstacle_at_cog_collides(pp):
    p = planner(pp, H=40)
    s = snapshot_towards(pp, (30, 0, 0, 0), 5.0, 40)
    s.obstacle_field = pp.extrapolate([pp.ObstaclePoint(0, 0, 0, 0)], 40, 0.1, pp.Pose2(0, 0, 0))
    r = p.rollout([0.5] * 18, s)
    assert r.collided and not r.reached


def test_zero_network_decelerates_straight(pp):
    p = planner(pp, H=10)
    r = p.rollout([0.0] * 18, snapshot_towards(pp, (1000, 0, 0, 10), 10.0, 10))
    assert (r.first_action.a0, r.first_action.a1) == (0.0, 0.0)
    assert abs(r.trajectory[1].x - 1.0) < 1e-12 and r.trajectory[1].y == 0.0
    assert abs(r.trajectory[1].v - 9.822190611664296) < 1e-12


@pytest.mark.parametrize("precision", [32, 64])
def test_evaluates_exact_budget(pp, precision):
    p = planner(pp, H=30, n_candidates=32, n_restarts=4, n_iter_max=2, precision=precision)
    out = p.plan_step(snapshot_towards(pp, (25, 0, 0, 5), 5.0, 30), 0)
    assert out.evaluated == 4 * 2 * 32


def test_early_exit_shortens_budget(pp):
    p = planner(pp, H=30, n_candidates=16, n_restarts=6, early_exit=True)
    out = p.plan_step(snapshot_towards(pp, (0, 0, 0, 0), 0.0, 30), 0)
    assert out.success and out.evaluated == 16


def test_degenerate_goal_keeps_warm_theta(pp):
    p = planner(pp, H=30, n_candidates=24, n_restarts=2)
    s = snapshot_towards(pp, (0, 0, 0, 0), 0.0, 30)
    s.warm_theta = [0.37] * 18
    out = p.plan_step(s, 0)
    assert out.success and out.predicted.t_goal == 0 and list(out.best_theta) == [0.37] * 18


def test_warm_start_dominance(pp):
    p = planner(pp, H=80, n_candidates=256, n_restarts=4, master_seed=17)
    first = snapshot_towards(pp, (8, 0, 0, 3), 3.0, 80)
    boot = p.plan_step(first, 0)
    assert boot.success
    warm = snapshot_towards(pp, (8, 0, 0, 3), 3.0, 80)
    warm.warm_theta = list(boot.best_theta)
    out = p.plan_step(warm, 1)
    assert not pp.better(pp.score(p.rollout(list(boot.best_theta), warm)), pp.score(out.predicted))


def test_more_restarts_never_score_worse(pp):
    rnd = np.random.default_rng(33)
    for trial in range(3):
        u = lambda: rnd.uniform(-1, 1)  # noqa: E731
        goal = (10 + 5 * u(), 3 * u(), 0.5 * u(), 2.0)
        s = snapshot_towards(pp, goal, 2.0 + u(), 60)
        small = planner(pp, H=60, n_candidates=48, n_restarts=1, master_seed=100 + trial,
                        precision=64)
        large = planner(pp, H=60, n_candidates=48, n_restarts=5, master_seed=100 + trial,
                        precision=64)
        assert not pp.better(pp.score(small.plan_step(s, 0).predicted),
                             pp.score(large.plan_step(s, 0).predicted))


def test_all_colliding_falls_back_to_braking(pp):
    p = planner(pp, H=20, n_candidates=32, n_restarts=2)
    s = snapshot_towards(pp, (20, 0, 0, 5), 5.0, 20)
    s.actuator = pp.ActuatorState(0.2)
    s.obstacle_field = pp.extrapolate([pp.ObstaclePoint(0, 0, 0, 0)], 20, 0.1, pp.Pose2(0, 0, 0))
    out = p.plan_step(s, 0)
    assert not out.success and out.predicted.collided
    assert out.action.a0 == 0.2 / pp.VehicleParams().delta_max and out.action.a1 == -1.0


def test_bit_identical_across_thread_counts(pp):
    s = snapshot_towards(pp, (15, 2, 0.3, 4), 5.3, 50)
    s.warm_theta = [0.1] * 18
    outs = [planner(pp, H=50, n_candidates=96, n_restarts=3, master_seed=5, threads=t)
            .plan_step(s, 7) for t in (1, 2, 8)]
    for o in outs[1:]:
        assert list(o.best_theta) == list(outs[0].best_theta)
        assert [z.x for z in o.predicted.trajectory] == [z.x for z in outs[0].predicted.trajectory]


def test_predicted_matches_independent_resimulation(pp):
    p = planner(pp, H=60, n_candidates=48, n_restarts=3, threads=2, master_seed=9)
    rnd = np.random.default_rng(35)
    for i in range(10):
        u = lambda: rnd.uniform(-1, 1)  # noqa: E731
        s = snapshot_towards(pp, (10 * u(), 8 * u(), PI * u(), 5 * u()), 6 * u(), 60)
        s.actuator = pp.ActuatorState(0.5 * u())
        s.prev_action = pp.ControlAction(u(), u())
        out = p.plan_step(s, i)
        resim = pp.resimulate_rollout(list(out.best_theta), s, p)
        assert (out.predicted.reached, out.predicted.collided, out.predicted.t_goal) == \
            (resim.reached, resim.collided, resim.t_goal)
        assert out.predicted.path_length == resim.path_length
        assert out.predicted.terminal_cost == resim.terminal_cost
        assert [(z.x, z.y, z.phi, z.v) for z in out.predicted.trajectory] == \
            [(z.x, z.y, z.phi, z.v) for z in resim.trajectory]


def test_prediction_collision_free_unless_fallback(pp):
    p = planner(pp, H=50, n_candidates=64, n_restarts=2)
    params = pp.VehicleParams()
    rnd = np.random.default_rng(36)
    for i in range(15):
        u = lambda: rnd.uniform(-1, 1)  # noqa: E731
        s = snapshot_towards(pp, (18 * u(), 10 * u(), PI * u(), 3.0), 4 + 3 * u(), 50)
        pts = [pp.ObstaclePoint(14 * u(), 8 * u(), PI * u(), 2 + 2 * u()) for _ in range(12)]
        s.obstacle_field = pp.extrapolate(pts, 50, 0.1, pp.Pose2(0, 0, 0))
        out = p.plan_step(s, i)
        if out.predicted.collided:
            assert not out.success and out.action.a1 == -1.0
        else:
            for h, z in enumerate(out.predicted.trajectory):
                assert not pp.collision(pp.Pose2(z.x, z.y, z.phi), s.obstacle_field.at(h), params)


def test_reference_smoke_small_closed_loop(pp):  # test_smoke.py:38-56
    spec = pp.builtin_scenario("exp2")
    c = spec.planner
    c.n_candidates, c.n_restarts = 24, 2
    m = spec.mission
    m.time_limit = 1.0
    log = pp.run_mission(m, c, spec.arch, 0)
    assert 1 <= len(log.records) <= 11 and log.stats.ticks <= 10
    rerun = pp.run_mission(m, c, spec.arch, 0)
    assert [r.state.x for r in rerun.records] == [r.state.x for r in log.records]


def test_reference_smoke_plan_step_degenerate_goal(pp):  # test_smoke.py:59-71
    p = planner(pp, H=20, n_candidates=8, n_restarts=1)
    s = pp.PlanningSnapshot()
    s.ev_state = pp.VehicleState(0, 0, 0, 0)
    s.goal = pp.GoalSetpoint(0, 0, 0, 0)
    s.obstacle_field = pp.extrapolate([], 20, 0.1, pp.Pose2(0, 0, 0))
    out = p.plan_step(s, 0)
    assert out.success and out.predicted.t_goal == 0


def test_selfchecks_pass(pp):
    res = pp.run_selfchecks()
    assert len(res) == 7
    assert all(r.pass_ for r in res), [(r.name, r.detail) for r in res if not r.pass_]


@pytest.mark.parametrize("precision", [64, 32])
def test_closed_loop_mission_vs_reference(pp, precision):
    """run_mission (Alg. 1) through the device planner vs the reference's
    own run_mission: identical per-tick records while the winners agree."""
    spec = pp.builtin_scenario("exp3_explicit")
    c = spec.planner
    c.H, c.n_candidates, c.n_restarts, c.precision = 30, 512, 2, precision
    m = spec.mission
    m.time_limit = 2.0
    log = pp.run_mission(m, c, spec.arch, 3)
    ref = Ref.lib()
    import ctypes as C
    rec = np.zeros((64, 8))
    tau = C.c_double()
    n = ref.ref_run_mission_builtin(b"exp3_explicit", 30, 512, 2, 2.0, 3, 1,
                                    rec.ctypes.data_as(C.POINTER(C.c_double)), 64, C.byref(tau))
    assert n == len(log.records)
    ours = np.array([[r.t, r.state.x, r.state.y, r.state.phi, r.state.v, r.action.a0,
                      r.action.a1, r.delta] for r in log.records])
    # certified winners (refine, the default) in FP32 as in FP64: every tick
    # is the reference's, bit for bit
    assert np.array_equal(ours, rec[:n])


def test_planner_config_extensions_exposed(pp):
    c = pp.PlannerConfig()
    assert c.precision == 32 and c.device == 0 and c.refine
    p = pp.Planner(pp.VehicleParams(), pp.MlpArchitecture([5, 2, 2]), c)
    assert p.device_handle != 0 and p.param_count == 18
    assert abi.Model().param_count() == 18


@pytest.mark.parametrize("precision", [32, 64])
def test_run_sweep_outputs_match_reference(pp, tmp_path, precision):
    """run_sweep (scenario.cpp:444-549) over the device planner writes the
    reference's files: scenario JSON, per-seed CSV / xy, report JSON --
    identical apart from the measured planning times."""
    import ctypes as C
    import json
    spec = pp.builtin_scenario("exp3_explicit")
    c = spec.planner
    c.H, c.n_candidates, c.n_restarts, c.precision = 30, 512, 2, precision
    spec.planner = c
    m = spec.mission
    m.time_limit = 1.5
    spec.mission = m
    spec.seeds = [3, 4]
    ours, ref = tmp_path / "ours", tmp_path / "ref"
    pp.run_sweep(spec, str(ours), 2)
    seeds = (C.c_uint64 * 2)(3, 4)
    assert Ref.lib().ref_run_sweep_builtin(b"exp3_explicit", 30, 512, 2, 1.5, seeds, 2, 2,
                                           str(ref).encode()) == 0
    names = sorted(p.name for p in ref.iterdir())
    assert names == sorted(p.name for p in ours.iterdir())

    def strip_tau(obj):
        if isinstance(obj, dict):
            return {k: strip_tau(v) for k, v in obj.items() if "tau" not in k}
        if isinstance(obj, list):
            return [strip_tau(v) for v in obj]
        return obj

    for name in names:
        a, b = (ours / name).read_text(), (ref / name).read_text()
        if name.endswith(".csv"):  # last column: measured plan time
            a = [ln.rsplit(",", 1)[0] for ln in a.splitlines()]
            b = [ln.rsplit(",", 1)[0] for ln in b.splitlines()]
            assert a == b, name
        elif name.endswith("_report.json"):
            assert strip_tau(json.loads(a)) == strip_tau(json.loads(b)), name
        else:  # scenario file (JSON with the reference's comments), xy files
            assert a == b, name


@pytest.mark.parametrize("precision", [32, 64])
def test_epilogue_reuses_certified_rollout_exactly(pp, precision):
    """The FP64 epilogue copies the certification's rollout of the final
    winner (capi.cpp, plan_step_resident) instead of re-simulating it: the
    copy must equal an independent re-simulation bit for bit, with obstacles,
    several restarts and hill-climb iterations (iter > 0 centres on the
    incumbent)."""
    H = 40
    p = planner(pp, H=H, n_candidates=4096, n_restarts=2, n_iter_max=3, precision=precision,
                master_seed=21)
    rnd = np.random.default_rng(77)
    for i in range(6):
        s = snapshot_towards(pp, (12 + 4 * rnd.uniform(), 3 * rnd.uniform(-1, 1), 0.3 * rnd.uniform(-1, 1),
                                  4.0), 5.0, H)
        obst = [pp.ObstaclePoint(6 + 2 * rnd.uniform(), rnd.uniform(-1.5, 1.5), rnd.uniform(-1, 1), 0.0)
                for _ in range(12)]
        s.obstacle_field = pp.extrapolate(obst, H, 0.1, pp.Pose2(0, 0, 0))
        out = p.plan_step(s, i)
        resim = pp.resimulate_rollout(list(out.best_theta), s, p)
        assert (out.predicted.reached, out.predicted.collided, out.predicted.t_goal) == \
            (resim.reached, resim.collided, resim.t_goal)
        assert out.predicted.path_length == resim.path_length
        assert out.predicted.terminal_cost == resim.terminal_cost
        assert (out.predicted.first_action.a0, out.predicted.first_action.a1) == \
            (resim.first_action.a0, resim.first_action.a1)
        assert [(z.x, z.y, z.phi, z.v) for z in out.predicted.trajectory] == \
            [(z.x, z.y, z.phi, z.v) for z in resim.trajectory]
