#!/usr/bin/env python
"""Benchmark of the per-control-step sampler (BASELINE.json metric).

Workload (N=1): configs[1] of BASELINE.json = C2, dynamic obstacle avoidance,
2^20 samples, horizon 30, 20 obstacle points (4 moving), NN-[5,2,2], FP32
rollout. With N GPUs (torchrun, one process per GPU) every
rank evaluates its own 2^20-candidate shard of an N x 2^20 candidate round
("weak" scaling) and the winner records are all-gathered over NCCL.

  value   sample-horizon-steps/s (samples * H / t), inputs resident in HBM,
          device time (CUDA events on the planner's stream) of each sampling
          round, max over ranks; L2 flushed between steps.
  e2e     the same metric through the public API (paraplan.Planner.plan_step
          at N=1, the sharded plan_step at N>1): host snapshot copied H2D,
          kernel, NCCL exchange, D2H and the FP64 host epilogue, wall clock.
  roofline  FP32 CUDA-core bound: algorithmic flops of the kernel
          (workloads.algorithmic_flops) / kernel time vs the FFMA peak measured
          on this GPU in the same run.
  cpu_baseline  the reference planner compiled from its own sources
          (oracle/_ref) on the host cores, bounded sample of the same workload.

--impl reference times only that CPU reference planner (all host threads).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sample_horizon_steps_per_s"
UNIT = "sample-horizon-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", type=int, default=32, choices=[32, 64])
    ap.add_argument("--samples", type=int, default=1 << 20, help="candidates per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="budget of the CPU-baseline sample")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_reference_timing(workload, cores: int, budget_s: float, steps: int | None = None,
                         warmup: int = 1):
    """The reference planner (oracle/_ref, compiled from its own sources) on a
    bounded sample of the workload: same snapshot, H and arch, fewer
    candidates. Returns (samples*H/s, sample description, per-step seconds)."""
    from oracle.oracle import Ref
    from paper_1904_06680_b200 import abi

    m0 = workload.model
    n = 1 << 14
    probe = abi.Model(H=m0.H, n_restarts=1, n_candidates=n, threads=cores)
    ref = Ref(probe)
    t0 = time.perf_counter()
    ref.plan_step(workload.snapshot, workload.t)
    dt = time.perf_counter() - t0
    # scale the sample so one step costs ~budget/4 (bounded by the workload)
    target = budget_s / (steps + warmup if steps else 4)
    n = int(min(m0.n_candidates, max(1 << 12, n * target / max(dt, 1e-6))))
    n = 1 << max(12, n.bit_length() - 1)
    model = abi.Model(H=m0.H, n_restarts=1, n_candidates=n, threads=cores)
    ref = Ref(model)
    for _ in range(warmup):
        ref.plan_step(workload.snapshot, workload.t)
    times = []
    reps = steps if steps else 3
    for _ in range(reps):
        t0 = time.perf_counter()
        ref.plan_step(workload.snapshot, workload.t)
        times.append(time.perf_counter() - t0)
    per = statistics.median(times)
    return n * m0.H / per, n, times


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1904_06680_b200 import workloads
    w = workloads.c2(samples=a.samples)
    cores = os.cpu_count() or 1
    value, n, times = cpu_reference_timing(w, cores, a.cpu_seconds * 4, steps=a.steps,
                                           warmup=max(1, min(a.warmup, 2)))
    ms = statistics.median(times) * 1e3
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 dynamic obstacle avoidance (bounded CPU sample)",
                   "samples": n, "H": w.model.H, "n_points": int(w.snapshot.field.shape[1]),
                   "arch": [5, 2, 2]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{n} of {w.samples} candidates of C2 per step, "
                                   f"reference Planner::plan_step threads={cores}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_b200(a):
    import torch

    from paper_1904_06680_b200 import abi, capi, import_paraplan, workloads
    from paper_1904_06680_b200.distributed import ShardedPlanner

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # more ranks than GPUs (a code-path check on a small box, not a measurement):
    # ranks share devices and exchange records over gloo (NCCL refuses two
    # ranks on one GPU)
    n_dev = torch.cuda.device_count()
    shared = world > n_dev
    local = local % max(n_dev, 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    per_gpu = a.samples
    w = workloads.c2(samples=per_gpu * world, precision=a.precision)
    model = w.model
    model.device = local
    H, N = model.H, int(w.snapshot.field.shape[1])

    peak_tf = None
    if rank == 0:
        peak_tf, _ = capi.measure_fp32_peak(local)

    # ---------------- value: device-resident sampling rounds -----------------
    from paper_1904_06680_b200.distributed import shard_range
    dp = capi.DevicePlanner(model)
    c0, c1 = shard_range(model.n_candidates, rank, world)
    dp.upload(w.snapshot)
    stream = torch.cuda.ExternalStream(dp.stream(), device=torch.device("cuda", local))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2
    center = np.zeros(model.param_count())
    for _ in range(a.warmup):
        dp.evaluate(None, w.t, 0, 0, 1, center, c0, c1)
    dev_ms, kern_ms, steps_exec, states, launches, refined = [], [], 0, 0, 0, 0
    barrier()
    with ClockSampler(local) as clocks:
        for _ in range(a.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dp.evaluate(None, w.t, 0, 0, 1, center, c0, c1)
            e1.record(stream)
            e1.synchronize()
            dev_ms.append(e0.elapsed_time(e1))
            tm = dp.timing()
            kern_ms.append(tm.kernel_ms)
            steps_exec += tm.executed_steps
            states += tm.checked_states
            launches += tm.launches
            refined += max(tm.refined, 0)
        barrier()
        total_ms = sum(dev_ms)
        if dist is not None:
            t = torch.tensor([total_ms], device="cpu" if shared else f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        value = model.n_candidates * H * a.steps / (total_ms * 1e-3)

        # ---------------- e2e: public API, host buffers ----------------------
        if world == 1:
            pp = import_paraplan()
            pc = pp.PlannerConfig()
            pc.H, pc.n_restarts, pc.n_candidates = H, 1, model.n_candidates
            pc.precision, pc.device, pc.n_obst_pts = a.precision, local, N
            planner = pp.Planner(pp.VehicleParams(), pp.MlpArchitecture([5, 2, 2]), pc)
            m = workloads.c2_mission()
            snap = pp.PlanningSnapshot()
            snap.ev_state = m.initial_state
            snap.prev_action = pp.ControlAction(0.0, pp.idle_longitudinal(pp.VehicleParams()))
            sel = pp.select_goal(m, m.initial_state, 0, pp.GoalTolerance())
            snap.goal = sel.goal
            ev = m.initial_state
            snap.obstacle_field = pp.extrapolate(pp.sense(m, ev, w.t, N, 0.1), H, 0.1,
                                                 pp.Pose2(ev.x, ev.y, ev.phi))
            handle = planner.device_handle

            def e2e_step():
                out = planner.plan_step(snap, w.t)
                return out.action.a0

            def e2e_timing():
                import ctypes as C
                tm = abi.pp_timing()
                capi.lib().pp_last_timing(C.c_void_p(handle), C.byref(tm))
                return tm
        else:
            sp = ShardedPlanner.on_device(model, rank, world)

            def e2e_step():
                return sp.plan_step(w.snapshot, w.t).action[0]

            def e2e_timing():
                return sp.device_planner.timing()

        for _ in range(a.warmup):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        h2d = d2h = 0
        for _ in range(a.steps):
            e2e_step()
            tm = e2e_timing()
            h2d += tm.h2d_bytes
            d2h += tm.d2h_bytes
        barrier()
        e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device="cpu" if shared else f"cuda:{local}",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = model.n_candidates * H * a.steps / e2e_s

    # ---------------- roofline ------------------------------------------------
    kern_avg_ms = sum(kern_ms) / len(kern_ms)
    flops = workloads.algorithmic_flops([5, 2, 2], N, steps_exec // a.steps, states // a.steps)
    achieved = flops / (kern_avg_ms * 1e-3) / 1e12
    traffic, traffic_live, pipes = None, None, None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        tj = json.loads(tf.read_text())
        traffic = tj.get("dram_bytes_per_launch")
        traffic_live = tj.get("live_dram_bytes_per_launch")
        pipes = tj.get("pipes")

    out = None
    if rank == 0:
        cpu = None
        if world == 1:
            cores = os.cpu_count() or 1
            cv, n_cpu, times = cpu_reference_timing(w, cores, a.cpu_seconds)
            cpu = {"value": cv, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"{n_cpu} of {w.samples} C2 candidates per plan_step, median of "
                             f"{len(times)}, reference Planner::plan_step threads={cores}"}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if a.precision == 32 else "f64", "data": "synthetic",
            "config": {"workload": "C2 dynamic obstacle avoidance (BASELINE.json configs[1])",
                       "samples_per_gpu": per_gpu, "samples_total": model.n_candidates,
                       "H": H, "n_points": N, "moving_points": 4, "arch": [5, 2, 2],
                       "restarts": 1, "parallelism": f"candidate shards x{world}",
                       "rollout_precision": "fp32" if a.precision == 32 else "fp64",
                       "winner": "certified: FP32 window re-ranked in the reference's FP64 "
                                 "arithmetic (PlannerConfig.refine)",
                       "l2": "flushed (256 MiB write) between timed steps",
                       **({"devices_shared": f"{world} ranks on {n_dev} GPU(s): code-path "
                                             "check only, not a scaling measurement"}
                          if shared else {})},
            "value_timing": "CUDA events on the planner stream around each sampling round "
                            "(generate + rollout + window-select kernels and the host "
                            "certification between them), snapshot resident in HBM",
            "near_tie_candidates_per_step": refined // a.steps,
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_s / a.steps * 1e3,
                    "h2d_bytes_per_step": h2d // a.steps, "d2h_bytes_per_step": d2h // a.steps,
                    "api": "paraplan.Planner.plan_step" if world == 1 else
                           "ShardedPlanner.plan_step (NCCL all-gather of winner records)"},
            "latency_ms": e2e_s / a.steps * 1e3,
            "gpu_launches": launches,
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": achieved / peak_tf if peak_tf else None,
                         "traffic": traffic, "traffic_live": traffic_live,
                         "peak_source": "FFMA loop measured in this run",
                         "ncu_pipes": pipes,
                         "kernel_ms": kern_avg_ms, "flops_per_launch": flops,
                         "executed_steps_per_launch": steps_exec // a.steps},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
