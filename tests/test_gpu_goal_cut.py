"""The goal-horizon cut (B200): rollouts of a restart stop a few states after
its earliest goal reach, and the certified plan stays the reference's.

A candidate that has not reached the goal by the restart's earliest t_goal T
plus the slack cannot win (src/planner.cpp:27-38 ranks class 2 first, then the
earliest t_goal), so the refill kernel stops its rollout there
(csrc/cuda/rollout.cuh, device_api.h kCutTGoal). The certificate accepts the
cut only when the exact best reaches by T + slack; otherwise the round is redone
without it (csrc/capi/round.cpp certify_round). Each case runs the planner in a
subprocess under one environment -- the cut on (default), off
(PARAPLAN_GOAL_CUT=0), and a negative slack that cuts rollouts before they
reach (PARAPLAN_CUT_SLACK=-6: the redo path) -- and compares the returned plan
with the CPU oracle's bit for bit.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.oracle import Port
from paper_1904_06680_b200 import workloads

pytestmark = pytest.mark.gpu
NPROC = os.cpu_count() or 1
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import json, sys
import numpy as np
from paper_1904_06680_b200 import capi, workloads
case, samples = sys.argv[1], int(sys.argv[2])
w = workloads.c4(samples=samples) if case == "c4" else workloads.c5(samples, 100, 1000)
dp = capi.DevicePlanner(w.model)
out, theta, traj = dp.plan_step(w.snapshot, w.t)
tm = dp.timing()
dp.close()
print(json.dumps(dict(candidate=int(out.winner.candidate), restart=int(out.winner.restart),
                      theta=[float(x) for x in theta], traj=np.asarray(traj).ravel().tolist(),
                      steps=int(tm.executed_steps), fp64_rounds=int(tm.fp64_rounds))))
"""


def run_child(case, samples, env_extra):
    env = dict(os.environ, PARAPLAN_TRACE="1", **env_extra)
    p = subprocess.run([sys.executable, "-c", _CHILD, case, str(samples)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1]), p.stderr


@pytest.mark.parametrize("case,samples", [("c4", 1 << 16), ("c5", 1 << 16)])
def test_goal_cut_plan_equals_oracle(case, samples):
    w = workloads.c4(samples=samples) if case == "c4" else workloads.c5(samples, 100, 1000)
    ref_out, ref_theta, ref_traj = Port(w.model).plan_step(w.snapshot, w.t, threads=NPROC)
    assert ref_out.winner.cls == 2  # a reaching winner: the cut applies
    runs = {}
    for name, env in [("cut", {}), ("off", {"PARAPLAN_GOAL_CUT": "0"}),
                      ("redo", {"PARAPLAN_CUT_SLACK": "-6"})]:
        res, err = run_child(case, samples, env)
        runs[name] = res
        assert res["candidate"] == ref_out.winner.candidate, (name, res["candidate"])
        assert np.array_equal(np.asarray(res["theta"]), ref_theta), name
        assert np.array_equal(np.asarray(res["traj"]), np.asarray(ref_traj).ravel()), name
        if name == "redo":
            assert "goal cut does not hold" in err, err[-2000:]
        else:
            assert "goal cut does not hold" not in err, (name, err[-2000:])
    # the cut skips states: fewer executed steps than running every rollout out
    assert runs["cut"]["steps"] < runs["off"]["steps"], (runs["cut"]["steps"], runs["off"]["steps"])
