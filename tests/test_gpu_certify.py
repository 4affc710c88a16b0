"""Certified re-ranking through its wide-window path (round.cpp certify_round):
windows wider than PARAPLAN_HOST_MAX go through the device FP64 list round
(generator + rollout over the listed members, with the goal cut when the
round has one restart) and the device pick filter (launch_list_filter) first,
and only the FP64 near-ties and FP64-flagged members to the host. The
returned plan must still be the reference's, bit for bit.

The window here is wide because many candidates reach a near goal on an
empty road at the same state index with path lengths within 0.1% (the C3
closed-loop situation); PARAPLAN_HOST_MAX=2 forces the device kernel even
for a small round. Runs in a subprocess: the knob is read once per process.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from oracle.oracle import Port
from paper_1904_06680_b200 import abi, capi

n, H, precision, gx = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
R = int(sys.argv[6])
snap = abi.Snapshot(ev=(0.0, 0.0, 0.0, 5.0), prev_action=(0.0, 0.32142857142857145),
                    goal=(gx, 0.0, 0.0, 5.0), field=np.zeros((H + 1, 0, 2)))
m = abi.Model(H=H, n_restarts=R, n_candidates=n, n_obst_pts=0, precision=precision)
o1, th1, tr1 = Port(m).plan_step(snap, 0)
dp = capi.DevicePlanner(m)
o2, th2, tr2 = dp.plan_step(snap, 0)
assert (o1.winner.restart, o1.winner.candidate) == (o2.winner.restart, o2.winner.candidate), \
    (o1.winner, o2.winner)
assert np.array_equal(th1, th2) and np.array_equal(tr1, tr2)
assert (o1.action_a0, o1.action_a1, o1.success) == (o2.action_a0, o2.action_a1, o2.success)
print("refined", dp.timing().refined, "cls", o2.winner.cls)
"""


# goal 2 m ahead at 5 m/s: ~100 candidates share the best state index with
# paths within 0.1%; 1.5 m: every candidate reaches at state 1 and the whole
# round (2 x 2^14) is one window
@pytest.mark.parametrize("restarts", [2, 1])
@pytest.mark.parametrize("gx", [2.0, 1.5])
@pytest.mark.parametrize("precision", [32, 64])
def test_wide_window_goes_through_device_fp64_and_returns_reference_plan(precision, gx, restarts):
    env = dict(os.environ, PARAPLAN_HOST_MAX="2", PARAPLAN_TRACE="1")
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), str(1 << 14), "120",
                        str(precision), str(gx), str(restarts)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "cls 2" in p.stdout, p.stdout  # the winner reaches the goal
    sel = [int(tok.split("=")[1]) for line in p.stderr.splitlines() if "pass=" in line
           for tok in line.split() if tok.startswith("selected=")]
    if precision == 32:  # the window went to the device FP64 list round and filter
        assert sel and max(sel) > 2, p.stderr
        assert "picked on the device" in p.stderr, p.stderr
