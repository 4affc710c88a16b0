"""The round's device time (pp_timing.kernel_ms): the θ generator stamps the
round's start (%globaltimer) into the round block and copy_out_kernel turns it
into the span up to the result store (csrc/cuda/rollout_f64.cu). It must
cover the rollout kernel's own span (rollout_ms, first CTA start to last CTA
end), fit inside CUDA events around the call, and be this round's alone (the
stamp is cleared for the next round)."""
from __future__ import annotations

import pytest
import torch

from paper_1904_06680_b200 import capi, workloads

pytestmark = pytest.mark.gpu


def test_round_span_covers_the_rollout_and_matches_events():
    w = workloads.c2(samples=1 << 18)
    dp = capi.DevicePlanner(w.model)
    dp.upload(w.snapshot)
    stream = torch.cuda.ExternalStream(dp.stream())
    for i in range(6):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dp.evaluate(None, w.t, 0, 0, 1, None, 0, w.model.n_candidates)
        e1.record(stream)
        e1.synchronize()
        ev_ms = e0.elapsed_time(e1)
        tm = dp.timing()
        assert 0.0 < tm.rollout_ms < tm.kernel_ms, (tm.rollout_ms, tm.kernel_ms)
        # the device span sits inside the events around the call (which also
        # hold the host's launches and certification), and it is this
        # round's: a stale start stamp would add whole rounds to it
        assert tm.kernel_ms <= ev_ms * 1.05 + 0.01, (tm.kernel_ms, ev_ms)
        assert tm.kernel_ms < tm.rollout_ms + 0.1, (tm.kernel_ms, tm.rollout_ms)
    dp.close()
