"""One C2 sampling round (2^20 candidates, H=30, 20 points) repeated --reps
times through the C-ABI: the command profiled under ncu (profiles/)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_06680_b200 import capi, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--precision", type=int, default=32)
ap.add_argument("--samples", type=int, default=1 << 20)
a = ap.parse_args()
w = workloads.c2(samples=a.samples, precision=a.precision)
dp = capi.DevicePlanner(w.model)
dp.upload(w.snapshot)
for _ in range(a.reps):
    rec, _ = dp.evaluate(None, w.t, 0, 0, 1, None, 0, w.model.n_candidates)
    t = dp.timing()
    print(f"kernel {t.kernel_ms:.3f} ms winner {rec[0]['candidate']} cls {rec[0]['cls']} "
          f"steps {t.executed_steps}")
