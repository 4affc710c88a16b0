"""Parked lanes (csrc/cuda/rollout.cuh refill_kernel): a rollout warp writes
its finished lanes' keys and refills them only every flush_every-th
iteration, and a parked lane must keep its final state until then
(step.cuh advance commits live lanes only). The per-candidate results may
not depend on the flush period: every candidate's rollout is the same
arithmetic whichever lane runs it and whenever its keys are written. Each
period runs in a subprocess (PARAPLAN_FLUSH_EVERY is read once per process)
and the per-sample outputs (class, t_goal, steps, path, terminal cost, first
action) must be identical bit for bit, in FP32 and FP64, on the C2 scene and
on a reaching scene, and so must the round winner (on the reaching scene from
the goal-cut variant with its waiting-lane rule; per-sample rounds run every
rollout to its end).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1904_06680_b200 import abi, capi, workloads
case, precision, out = sys.argv[2], int(sys.argv[3]), sys.argv[4]
if case == "c2":
    w = workloads.c2(samples=1 << 16, precision=precision)
    snap, t, m = w.snapshot, w.t, w.model
else:  # a near goal on an empty road: the winner reaches (cut variant)
    H = 60
    snap = abi.Snapshot(ev=(0.0, 0.0, 0.0, 5.0), prev_action=(0.0, 0.32142857142857145),
                        goal=(8.0, 0.0, 0.0, 5.0), field=np.zeros((H + 1, 0, 2)))
    t = 0
    m = abi.Model(H=H, n_restarts=1, n_candidates=1 << 16, n_obst_pts=0, precision=precision)
m.refine = 0
dp = capi.DevicePlanner(m)
n = m.n_candidates
dp.evaluate(snap, t, 0, 0, 1, None, 0, n)  # a first round sets the flush rule
rec, _ = dp.evaluate(snap, t, 0, 0, 1, None, 0, n)  # (reaching: the goal-cut variant)
_, ps = dp.evaluate(snap, t, 0, 0, 1, None, 0, n, per_sample=True)
np.save(out, ps)
np.save(out + ".win.npy", np.array([rec[0]["cls"], rec[0]["candidate"], rec[0]["k1"], rec[0]["k2"]]))
"""


def run(case, precision, period, tmp):
    out = tmp / f"{case}_{precision}_{period}.npy"
    env = dict(os.environ)
    if period:
        env["PARAPLAN_FLUSH_EVERY"] = str(period)
    else:
        env.pop("PARAPLAN_FLUSH_EVERY", None)
    p = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), case, str(precision), str(out)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return np.load(out), np.load(str(out) + ".win.npy")


@pytest.mark.parametrize("case", ["c2", "reach"])
@pytest.mark.parametrize("precision", [32, 64])
def test_per_sample_results_do_not_depend_on_the_flush_period(case, precision, tmp_path):
    ref, win = run(case, precision, 1, tmp_path)   # flush every iteration
    for period in (0, 4):                          # 0: the host's rule
        got, gwin = run(case, precision, period, tmp_path)
        for k in ref.dtype.names:
            assert np.array_equal(got[k], ref[k]), (case, precision, period, k)
        assert np.array_equal(gwin, win), (case, precision, period, gwin, win)
    if case == "reach":  # the winner reaches: the rounds after the first run the cut variant
        assert win[0] == 2 and ref["reached"].any()
