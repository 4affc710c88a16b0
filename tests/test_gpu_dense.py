"""Dense obstacle clouds: the 2-D cell grid, static-row dedup, early exit and
the host cell index must give the reference's verdicts exactly (the oracle
scans every point of every row)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle.oracle import Port
from paper_1904_06680_b200 import abi, capi, workloads

pytestmark = pytest.mark.gpu


def _plan_equal(w):
    o1, th1, tr1 = Port(w.model).plan_step(w.snapshot, w.t)
    o2, th2, tr2 = capi.DevicePlanner(w.model).plan_step(w.snapshot, w.t)
    assert np.array_equal(th1, th2) and np.array_equal(tr1, tr2)
    assert (o1.action_a0, o1.action_a1, o1.success) == (o2.action_a0, o2.action_a1, o2.success)


@pytest.mark.parametrize("n_points", [200, 1000])
@pytest.mark.parametrize("precision", [32, 64])
def test_c5_cloud_plan_matches_oracle(n_points, precision):
    w = workloads.c5(4096, 30, n_points, precision=precision)
    _plan_equal(w)


def test_c4_lot_plan_matches_oracle():
    w = workloads.c4(samples=2048, H=60)
    _plan_equal(w)


@pytest.mark.parametrize("precision", [32, 64])
def test_c4_lot_per_sample_stats(precision):
    w = workloads.c4(samples=1024, H=40, precision=precision)
    w.model.refine = 0
    dp = capi.DevicePlanner(w.model)
    _, got = dp.evaluate(w.snapshot, w.t, 0, 0, 1, None, 0, 1024, per_sample=True)
    want = Port(w.model).eval_candidates(w.snapshot, w.t, 0, 0, np.zeros(18), 0, 1024)
    flips = np.count_nonzero(got["collided"] != want["collided"])
    assert flips <= (0 if precision == 64 else 5)
    same = got["steps"] == want["steps"]
    assert same.mean() >= 0.99


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("which", ["c2", "c5_mixed", "c5_static", "c5_dense", "c4_lot"])
def test_raw_points_path_equals_extrapolated_field(which, precision):
    """pp_plan_step_points(points) == pp_plan_step(extrapolate(points)),
    bit for bit (the field is built by the planner; c5_dense
    bins its movers on the device, c4_lot uses the cell-box grid mode)."""
    import math
    rng = np.random.default_rng(7)
    if which == "c2":
        w = workloads.c2(samples=1 << 14, precision=precision)
        from paper_1904_06680_b200 import import_paraplan
        pp = import_paraplan()
        m = workloads.c2_mission()
        pts = np.array([(q.x, q.y, q.heading, q.speed)
                        for q in pp.sense(m, m.initial_state, w.t, 20, 0.1)])
    elif which == "c4_lot":
        w = workloads.c4(samples=1 << 13, H=60, precision=precision)
        pts = w.extra["points"]
    else:
        n = 10000 if which == "c5_dense" else 500  # c5_dense: movers binned on the device
        pts = np.zeros((n, 4))
        pts[:, 0] = rng.uniform(-10, 30, n)
        pts[:, 1] = rng.uniform(2.5, 10, n) * rng.choice([-1, 1], n)
        if which in ("c5_mixed", "c5_dense"):
            dyn = rng.random(n) < 0.25
            pts[dyn, 2] = rng.choice([0.0, math.pi], dyn.sum())
            pts[dyn, 3] = rng.uniform(0, 15, dyn.sum())
        w = workloads.c5(1 << 14, 30, n, precision=precision)
    snap = abi.Snapshot(ev=w.snapshot.ev, actuator_delta=w.snapshot.actuator_delta,
                        prev_action=w.snapshot.prev_action, goal=w.snapshot.goal,
                        field=abi.extrapolate(pts, w.model.H))
    dp = capi.DevicePlanner(w.model)
    o1, th1, tr1 = dp.plan_step(snap, w.t)
    o2, th2, tr2 = dp.plan_step_points(snap, pts, w.t)
    assert np.array_equal(th1, th2) and np.array_equal(tr1, tr2)
    assert (o1.action_a0, o1.action_a1, o1.evaluated) == (o2.action_a0, o2.action_a1, o2.evaluated)
    if which != "c4_lot":  # the lot at H=60 is too slow for the CPU oracle here
        o3, th3, tr3 = Port(w.model).plan_step(snap, w.t)
        assert np.array_equal(th1, th3) and np.array_equal(tr1, tr3)


def test_raw_points_errors_and_edge_cases():
    """pp_plan_step_points: non-finite points are rejected with the reference's
    message; no points and all-static points plan like the field path."""
    w = workloads.c5(1 << 12, 20, 100)
    pts = w.extra["points"].copy()
    dp = capi.DevicePlanner(w.model)
    bad = pts.copy()
    bad[3, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        dp.plan_step_points(w.snapshot, bad, w.t)
    # the planner stays usable after the error
    for sub in (pts[:0], pts[pts[:, 3] == 0], pts):
        snap = abi.Snapshot(ev=w.snapshot.ev, actuator_delta=w.snapshot.actuator_delta,
                            prev_action=w.snapshot.prev_action, goal=w.snapshot.goal,
                            field=abi.extrapolate(sub, w.model.H) if len(sub) else None)
        o1, th1, tr1 = dp.plan_step(snap, w.t)
        o2, th2, tr2 = dp.plan_step_points(snap, sub, w.t)
        assert np.array_equal(th1, th2) and np.array_equal(tr1, tr2)
        assert o1.evaluated == o2.evaluated


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("n, movers", [(12, False), (40, True), (100, True), (100, False)])
def test_small_fields_every_kernel_kind(n, movers, precision):
    """Small clouds on the road ahead, one per rollout kernel kind: all-static
    and all-dynamic x-buckets staged in shared memory with one part (kind 3;
    <= 64 points with a mover are made all-dynamic), and a mixed cloud of 100
    points (x-buckets with both parts, kind 0). The plan must be the oracle's."""
    import math
    rng = np.random.default_rng(n + (1000 if movers else 0))
    pts = np.zeros((n, 4))
    pts[:, 0] = rng.uniform(4.0, 30.0, n)
    pts[:, 1] = rng.uniform(-3.5, 3.5, n)
    if movers:
        dyn = rng.random(n) < 0.3
        pts[dyn, 2] = rng.choice([0.0, math.pi, 0.5 * math.pi], dyn.sum())
        pts[dyn, 3] = rng.uniform(0.0, 8.0, dyn.sum())
    w = workloads.c5(1 << 13, 30, n, precision=precision)
    snap = abi.Snapshot(ev=w.snapshot.ev, actuator_delta=w.snapshot.actuator_delta,
                        prev_action=w.snapshot.prev_action, goal=w.snapshot.goal,
                        field=abi.extrapolate(pts, w.model.H))
    w.snapshot = snap
    _plan_equal(w)


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_tiny_fields_scan_group_overrun(n, precision):
    """Kind 3 scans whole groups of kK3Group points (device_api.h): the last
    group of the warp's longest window reads past it, into points further in
    x or into the sentinel padding (N + kK3Group - 1 sentinels after the
    part). Tiny all-static clouds right on the road, odd and even N, so that
    windows end at the image's last point: every rollout's outcome must be
    the oracle's (FP64 exactly; FP32 within the flip budget of the other
    per-sample tests), and the certified plan equal."""
    rng = np.random.default_rng(77 + n)
    pts = np.zeros((n, 4))
    pts[:, 0] = rng.uniform(5.0, 15.0, n)
    pts[:, 1] = rng.uniform(-1.0, 1.0, n)
    w = workloads.c5(2048, 30, n, precision=precision)
    w.snapshot = abi.Snapshot(ev=w.snapshot.ev, actuator_delta=w.snapshot.actuator_delta,
                              prev_action=w.snapshot.prev_action, goal=w.snapshot.goal,
                              field=abi.extrapolate(pts, w.model.H))
    _plan_equal(w)
    w.model.refine = 0
    dp = capi.DevicePlanner(w.model)
    _, got = dp.evaluate(w.snapshot, w.t, 0, 0, 1, None, 0, 2048, per_sample=True)
    want = Port(w.model).eval_candidates(w.snapshot, w.t, 0, 0, np.zeros(18), 0, 2048)
    assert want["collided"].any()  # the cloud is in the way
    flips = np.count_nonzero(got["collided"] != want["collided"])
    assert flips <= (0 if precision == 64 else 5)
    if precision == 64:
        assert np.array_equal(got["steps"], want["steps"])
