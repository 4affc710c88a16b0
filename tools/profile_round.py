"""One sampling round (default C2 (2^20 candidates, H=30, 20 points) repeated --reps
times through the C-ABI: the command profiled under ncu (profiles/)."""
import argparse
import os
import sys
from pathlib import Path

# the construction warm-up round would be the first launches ncu captures
os.environ.setdefault("PARAPLAN_PREWARM", "0")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_06680_b200 import capi, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--precision", type=int, default=32)
ap.add_argument("--samples", type=int, default=1 << 20)
ap.add_argument("--refine", type=int, default=1)
ap.add_argument("--workload", default="c2", help="c2 | c4 | c5:N:H")
a = ap.parse_args()
if a.workload == "c2":
    w = workloads.c2(samples=a.samples, precision=a.precision)
elif a.workload == "c4":
    w = workloads.c4(samples=a.samples, precision=a.precision)
else:
    _, n_pts, H = a.workload.split(":")
    w = workloads.c5(a.samples, int(H), int(n_pts), precision=a.precision)
w.model.refine = a.refine
dp = capi.DevicePlanner(w.model)
dp.upload(w.snapshot)
import time  # noqa: E402
for _ in range(a.reps):
    t0 = time.perf_counter()
    rec, _ = dp.evaluate(None, w.t, 0, 0, 1, None, 0, w.model.n_candidates)
    wall = (time.perf_counter() - t0) * 1e3
    t = dp.timing()
    print(f"p{a.precision} refine={a.refine} wall {wall:.3f} ms device {t.kernel_ms:.3f} ms winner "
          f"{rec[0]['candidate']} cls {rec[0]['cls']} k1 {rec[0]['k1']:.12f} "
          f"steps {t.executed_steps} refined {t.refined} launches {t.launches} "
          f"certify {t.certify_ms:.3f} ms")
