"""The drop-in module's host primitives, restating the reference's unit tests
(/root/reference/proj/tests/{dynamics,geometry,policy,planner}_test.cpp and
tests/python/test_smoke.py) against `paraplan._core` built from this repo.
CPU-only: nothing here launches a kernel."""
from __future__ import annotations

import math

import pytest

PI = math.pi


def test_param_counts(pp):  # policy_test.cpp:13-17, test_smoke.py
    assert pp.param_count(pp.MlpArchitecture([5, 2, 2])) == 18
    assert pp.param_count(pp.MlpArchitecture([5, 10, 2])) == 82
    assert pp.param_count(pp.MlpArchitecture([5, 10, 10, 2])) == 192


@pytest.mark.parametrize("sizes", [[5], [4, 2, 2], [5, 2, 3], [5, 0, 2], [5, 257, 2]])
def test_architecture_validation(pp, sizes):  # policy_test.cpp:19-28
    with pytest.raises(ValueError):
        pp.MlpArchitecture(sizes)
    pp.MlpArchitecture([5, 7, 7, 2])


def test_idle_longitudinal(pp):  # dynamics_test.cpp:120-134, test_smoke.py
    p = pp.VehicleParams()
    idle = pp.idle_longitudinal(p)
    assert abs(idle - 0.321429) < 1e-6
    assert abs(pp.map_controls(pp.ControlAction(0.0, idle), pp.ActuatorState(0.0), p).u_v) < 1e-12


def test_map_controls_known_answers(pp):  # dynamics_test.cpp:13-58
    p = pp.VehicleParams()
    u = pp.map_controls(pp.ControlAction(0.0, pp.idle_longitudinal(p)), pp.ActuatorState(0.0), p)
    assert u.delta == 0.0
    u = pp.map_controls(pp.ControlAction(1.0, 1.0), pp.ActuatorState(0.0), p)
    assert abs(u.delta - 0.0349065850398866) < 1e-12
    assert u.u_v == p.u_v_max and abs(u.u_v - 3.7537537537537538) < 1e-12
    u = pp.map_controls(pp.ControlAction(-1.0, -1.0), pp.ActuatorState(-0.7), p)
    assert abs(u.delta - (-0.6981317007977318)) < 1e-12
    assert u.u_v == p.u_v_min and abs(u.u_v - (-7.309941520467836)) < 1e-12
    assert pp.map_controls(pp.ControlAction(0.0, -7.0), pp.ActuatorState(0.0), p).u_v == p.u_v_min
    assert pp.map_controls(pp.ControlAction(9.0, 7.0), pp.ActuatorState(0.0), p).u_v == p.u_v_max
    window = p.delta_rate_max * p.T_s
    for a0 in (-3.0, -0.4, 0.0, 0.6, 2.0):
        for d in (-0.7, -0.1, 0.3):
            c = pp.map_controls(pp.ControlAction(a0, 0.0), pp.ActuatorState(d), p)
            assert abs(c.delta - d) <= window + 1e-12 and abs(c.delta) <= p.delta_max


def test_euler_step_known_answers(pp):  # dynamics_test.cpp:60-93, test_smoke.py
    p = pp.VehicleParams()
    z = pp.step(pp.VehicleState(0, 0, 0, 10), 0.0, 0.0, p)
    assert (z.x, z.y, z.phi, z.v) == (1.0, 0.0, 0.0, 10.0)
    z = pp.step(pp.VehicleState(2.0, -3.0, 0.7, 0.0), p.delta_max, 0.0, p)
    assert (z.x, z.y, z.phi, z.v) == (2.0, -3.0, 0.7, 0.0)
    z = pp.step(pp.VehicleState(0, 0, 0, 1.0), p.delta_max, 0.0, p)
    assert abs(z.phi - 0.0335639852470912) < 1e-12
    z = pp.VehicleState(0, 0, 0, 0)
    for _ in range(10):
        z = pp.step(z, 0.0, p.u_v_min, p)
    assert z.v < 0 and z.x < 0


def test_vehicle_params_validation(pp):  # dynamics_test.cpp:136-148
    for field, value in (("l_f", 0.0), ("delta_max", 2.0), ("u_v_min", 1.0), ("T_s", 0.0)):
        p = pp.VehicleParams()
        setattr(p, field, value)
        with pytest.raises(ValueError):
            p.validate()
    pp.VehicleParams().validate()


def test_wrap_angle(pp):  # geometry_test.cpp:14-21
    assert abs(pp.wrap_angle(350.0 * PI / 180.0) - (-10.0 * PI / 180.0)) < 1e-12
    assert pp.wrap_angle(0.0) == 0.0
    assert abs(pp.wrap_angle(PI) - PI) < 1e-12
    assert abs(pp.wrap_angle(-PI) - PI) < 1e-12
    assert abs(pp.wrap_angle(3.0 * PI) - PI) < 1e-12
    assert abs(pp.wrap_angle(-5.5 * PI) - 0.5 * PI) < 1e-12


def test_frames(pp):  # geometry_test.cpp:23-50
    p = pp.to_ev_frame(pp.Pose2(0, 0, 0), pp.Vec2(3.0, 4.0))
    assert (p.x, p.y) == (3.0, 4.0)
    q = pp.from_ev_frame(pp.Pose2(0, 0, 0), pp.Vec2(3.0, 4.0))
    assert (q.x, q.y) == (3.0, 4.0)
    p = pp.to_ev_frame(pp.Pose2(1.0, 1.0, PI / 2), pp.Vec2(1.0, 2.0))
    assert abs(p.x - 1.0) < 1e-12 and abs(p.y) < 1e-12


def test_collision_boundaries(pp):  # geometry_test.cpp:52-90, test_smoke.py
    o = pp.Pose2(0, 0, 0)
    assert pp.collision(o, [pp.Vec2(0, 0)])
    assert not pp.collision(o, [pp.Vec2(1.9, 0)])
    assert not pp.collision(o, [pp.Vec2(1.8, 0)])   # front face: strict
    assert not pp.collision(o, [pp.Vec2(-2.0, 0)])  # rear face
    assert not pp.collision(o, [pp.Vec2(0, 1.0)])   # side
    assert pp.collision(o, [pp.Vec2(1.7999, 0)])
    assert not pp.collision(o, [])


def test_collision_matches_polygon_oracle(pp):  # acceptance criterion 3 (1e4 pairs)
    import random
    rnd = random.Random(12)
    p = pp.VehicleParams()
    tested = bad = 0
    for _ in range(10000):
        pose = pp.Pose2(rnd.uniform(-10, 10), rnd.uniform(-10, 10), rnd.uniform(-4 * PI, 4 * PI))
        pt = pp.Vec2(pose.x + rnd.uniform(-4, 4), pose.y + rnd.uniform(-4, 4))
        want = pp.chassis_oracle(pose, pt, p)
        if want is None:
            continue
        tested += 1
        bad += pp.collision(pose, [pt], p) != want
    assert bad == 0 and tested > 9000


def test_extrapolate(pp):  # geometry_test.cpp:52-93
    f = pp.extrapolate([pp.ObstaclePoint(5.0, 0.0, PI, 20.0 / 3.6)], 5, 0.1, pp.Pose2(0, 0, 0))
    assert f.n_points == 1
    assert abs(f.at(2)[0].x - 3.888888888888889) < 1e-12 and abs(f.at(2)[0].y) < 1e-12
    f = pp.extrapolate([pp.ObstaclePoint(1.5, -2.0, 0.7, 0.0)], 10, 0.1, pp.Pose2(0, 0, 0))
    assert all((f.at(h)[0].x, f.at(h)[0].y) == (1.5, -2.0) for h in range(11))
    empty = pp.extrapolate([], 7, 0.1, pp.Pose2(0, 0, 0))
    assert empty.n_points == 0 and all(empty.at(h) == [] for h in range(8))


def test_policy_forward(pp):  # policy_test.cpp:30-90, test_smoke.py
    pol = pp.MlpPolicy(pp.MlpArchitecture([5, 2, 2]))
    a = pol.forward([0.0] * pol.param_count, [0.3, -0.7, 0.1, 0.9, -0.2])
    assert (a.a0, a.a1) == (0.0, 0.0)
    theta = [0.0] * 18
    theta[0] = 1.0   # W1[0][0]
    theta[12] = 1.0  # W2[0][0]
    a = pol.forward(theta, [1.0, 0, 0, 0, 0])
    assert abs(a.a0 - 0.6420149920119997) < 1e-12 and a.a1 == 0.0
    with pytest.raises(ValueError):
        pol.forward([0.0] * 17, [0, 0, 0, 0, 0])


def test_build_features(pp):  # policy_test.cpp:92-116
    nc = pp.NormConstants()
    s = pp.build_features(pp.VehicleState(0, 0, 0, 0), pp.GoalSetpoint(0, 0, 0, 0), 0.3, nc)
    assert list(s) == [0.0, 0.0, 0.0, 0.0, 0.3]
    s = pp.build_features(pp.VehicleState(0, 0, 0, 0), pp.GoalSetpoint(30.0, 0, 0, 0), 0.0, nc)
    assert abs(s[0] - 1.0) < 1e-12
    s = pp.build_features(pp.VehicleState(0, 0, 0, 0), pp.GoalSetpoint(0, 0, 350 * PI / 180, 0),
                          0.0, nc)
    assert abs(s[2] - (-0.027777777777777776)) < 1e-12


def test_score_ordering():  # planner_test.cpp:34-51 via the C-ABI comparator
    from paper_1904_06680_b200 import capi
    better = capi.lib().pp_key_better
    assert better(2, -50.0, -30.0, 2, -80.0, -10.0) == 1   # earlier goal entry wins
    assert better(2, -80.0, -10.0, 2, -50.0, -30.0) == 0
    assert better(1, -99.0, 0.0, 0, -0.01, 0.0) == 1       # free beats collided
    assert better(2, -50.0, -20.0, 2, -50.0, -25.0) == 1   # shorter path breaks ties
    assert better(1, -1.0, 0.0, 1, -1.0, 0.0) == 0         # strict


def test_planner_config_validation(pp):  # planner_test.cpp:313-327
    for field, value in (("n_candidates", 0), ("H", 0), ("n_restarts", 0), ("threads", 0),
                         ("precision", 16)):
        c = pp.PlannerConfig()
        setattr(c, field, value)
        with pytest.raises(ValueError):
            c.validate()
    c = pp.PlannerConfig()
    c.sigma_log_low, c.sigma_log_high = 2.0, 1.0
    with pytest.raises(ValueError):
        c.validate()
    pp.PlannerConfig().validate()


def test_builtin_scenarios(pp, tmp_path):  # test_smoke.py, scenario_test.cpp
    names = pp.builtin_scenario_names()
    assert len(names) == 7
    assert pp.builtin_scenario("exp1").mission.waypoints[0].phi == PI
    with pytest.raises(pp.UsageError):
        pp.builtin_scenario("nope")
    for n in names:
        spec = pp.builtin_scenario(n)
        f = tmp_path / f"{n}.json"
        pp.save_scenario(spec, str(f))
        back = pp.load_scenario(str(f))
        assert pp.serialize_scenario(back) == pp.serialize_scenario(spec)


def test_serialized_scenarios_match_reference_text(pp):
    """serialize_scenario (scenario.cpp:204-266) writes the reference's text,
    provenance comments included, for every builtin scenario."""
    import ctypes as C
    from oracle.oracle import Ref
    for n in pp.builtin_scenario_names():
        buf = C.create_string_buffer(1 << 20)
        size = Ref.lib().ref_serialize_builtin(n.encode(), buf, len(buf))
        assert 0 < size < len(buf)
        assert pp.serialize_scenario(pp.builtin_scenario(n)) == buf.value.decode(), n


def test_no_gpu_fails_loudly(pp):
    """Without a device the planner must refuse, never fall back to the CPU."""
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pp.Planner(pp.VehicleParams(), pp.MlpArchitecture([5, 2, 2]), pp.PlannerConfig())
