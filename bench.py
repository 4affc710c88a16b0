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
    ap.add_argument("--allow-shared", action="store_true",
                    help="allow more ranks than GPUs (code-path check, not a measurement)")
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


def bench_config(a, world: int) -> dict:
    """The workload identity, shared by both arms (the driver compares them)."""
    return {"workload": "C2 dynamic obstacle avoidance (BASELINE.json configs[1])",
            "samples_per_gpu": a.samples, "samples_total": a.samples * world, "H": 30,
            "n_points": 20, "moving_points": 4, "arch": [5, 2, 2], "restarts": 1,
            "parallelism": f"candidate shards x{world}"}


def c2_reference_snapshot():
    """The C2 snapshot built by the REFERENCE's own select_goal -> sense ->
    extrapolate (oracle/_ref), so the reference arm never loads this repo's
    native code (workloads.c2_mission_arrays is plain data)."""
    from oracle.oracle import Ref
    from paper_1904_06680_b200 import workloads as W
    wp, st, dy, ev = W.c2_mission_arrays()
    return Ref.mission_snapshot(wp, st, dy, ev, W.C2_T, W.C2_H, W.C2_N_OBST), W.C2_T, W.C2_H


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


def thread_counts(nproc: int) -> list[int]:
    out, k = [], 1
    while k < nproc:
        out.append(k)
        k *= 2
    return out + [nproc]


def spin_calibration(nproc: int) -> dict:
    """W threads x 2.5 ms of independent spin work, wall
    time (raw std::thread and the reference's own ThreadPool)."""
    from oracle.oracle import Ref
    L = Ref.lib()
    rows = []
    for w in thread_counts(nproc):
        raw = min(L.ref_spin_calibration(w, 2.5, 0) for _ in range(3))
        pool = min(L.ref_spin_calibration(w, 2.5, 1) for _ in range(3))
        rows.append({"threads": w, "raw_ms": round(raw, 3), "pool_ms": round(pool, 3),
                     "efficiency": round(2.5 / pool, 3)})
    return {"work_per_thread_ms": 2.5, "rows": rows}


def cpu_protocol(snap, t: int, H: int, total: int, budget_s: float) -> dict:
    """The reference planner (oracle/_ref, compiled from its own sources) on
    the box's host cores: spin calibration, then a thread
    sweep {1, 2, 4, ..., nproc} of Planner::plan_step on a bounded sample of
    the workload (same snapshot, H and arch, fewer candidates), 1 warm-up +
    best / median of the timed calls."""
    from oracle.oracle import Ref
    from paper_1904_06680_b200 import abi
    nproc = os.cpu_count() or 1
    counts = thread_counts(nproc)
    # size the sample: one single-thread call ~ budget / (3 * len(counts))
    probe = Ref(abi.Model(H=H, n_restarts=1, n_candidates=2048, threads=1))
    t0 = time.perf_counter()
    probe.plan_step(snap, t)
    per_cand = (time.perf_counter() - t0) / 2048
    n = int(min(total, max(4096, budget_s / (3 * len(counts)) / max(per_cand, 1e-9))))
    n = 1 << (n.bit_length() - 1)
    sweep = []
    for th in counts:
        ref = Ref(abi.Model(H=H, n_restarts=1, n_candidates=n, threads=th))
        ref.plan_step(snap, t)  # warm-up (pool threads spawned)
        reps = 5 if th == nproc else 2
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            ref.plan_step(snap, t)
            times.append(time.perf_counter() - t0)
        sweep.append({"threads": th, "best_ms": round(min(times) * 1e3, 3),
                      "median_ms": round(statistics.median(times) * 1e3, 3),
                      "steps_per_s": n * H / min(times)})
    best = max(sweep, key=lambda r: r["steps_per_s"])
    at_nproc = sweep[-1]
    return {"value": best["steps_per_s"], "unit": UNIT, "cores": best["threads"],
            "kind": "reference", "nproc": nproc, "cpu_model": cpu_model(),
            "value_at_nproc": at_nproc["steps_per_s"],
            "sample": f"{n} of {total} C2 candidates (same snapshot, H, arch) per "
                      f"reference Planner::plan_step; 1 warm-up, best of 2-5 calls per "
                      f"thread count; value = best thread count ({best['threads']})",
            "thread_sweep": sweep, "spin_calibration": spin_calibration(nproc)}


def run_reference(a):
    """--impl reference: the unmodified reference planner (oracle/_ref) on
    the host cores, all threads, on the same C2 workload; only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.oracle import Ref
    from paper_1904_06680_b200 import abi
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    snap, t, H = c2_reference_snapshot()
    total = a.samples * world
    proto = cpu_protocol(snap, t, H, total, budget_s=a.cpu_seconds)
    nproc = proto["nproc"]
    # timed steps: all host threads, a sample sized so the K + W calls take
    # about 4 x cpu_seconds
    at = proto["thread_sweep"][-1]
    n_s = int(proto["sample"].split(" of ")[0])
    per_call = at["best_ms"] * 1e-3 / n_s
    n = int(min(total, max(4096, 4 * a.cpu_seconds / (a.steps + a.warmup) / max(per_call, 1e-9))))
    n = 1 << (n.bit_length() - 1)
    ref = Ref(abi.Model(H=H, n_restarts=1, n_candidates=n, threads=nproc))
    for _ in range(max(1, a.warmup)):
        ref.plan_step(snap, t)
    times = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        ref.plan_step(snap, t)
        times.append(time.perf_counter() - t0)
    per = statistics.median(times)
    value = n * H / per
    cpu = dict(proto)
    cpu.update({"value": value, "cores": nproc,
                "sample": f"{n} of {total} C2 candidates per reference Planner::plan_step "
                          f"(same snapshot, H, arch), threads={nproc}, median of {a.steps}"})
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(a, world),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def spawn_ranks(a) -> int:
    """`bench.py --gpus N` without torchrun: launch N ranks (one per GPU) the
    way the driver does, after checking that N GPUs exist."""
    import torch
    n_dev = torch.cuda.device_count()
    if n_dev < a.gpus and not a.allow_shared:
        print(json.dumps({"error": f"--gpus {a.gpus} but only {n_dev} CUDA device(s) visible"}),
              flush=True)
        return 2
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.call(cmd)


def run_b200(a):
    import torch

    from paper_1904_06680_b200 import abi, capi, import_paraplan, workloads
    from paper_1904_06680_b200.distributed import ShardedPlanner, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_dev = torch.cuda.device_count()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    # more ranks than GPUs only on request (a code-path check on a small box,
    # never a measurement): ranks share devices and exchange over gloo
    shared = world > n_dev
    if shared and not a.allow_shared:
        raise SystemExit(f"{world} ranks but only {n_dev} CUDA device(s); "
                         "--allow-shared runs a code-path check, not a measurement")
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

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], device="cpu" if shared else f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    per_gpu = a.samples
    w = workloads.c2(samples=per_gpu * world, precision=a.precision)
    model = w.model
    model.device = local
    H, N = model.H, int(w.snapshot.field.shape[1])

    peak_tf = None
    if rank == 0:
        peak_tf, _ = capi.measure_fp32_peak(local)

    # ---------------- value: device-resident sampling rounds -----------------
    dp = capi.DevicePlanner(model)
    dp.upload(w.snapshot)
    stream = torch.cuda.ExternalStream(dp.stream(), device=torch.device("cuda", local))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2

    def device_rounds(c0, c1, steps, stats=None):
        """`steps` sampling rounds over [c0, c1); returns the device ms of each."""
        out = []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dp.evaluate(None, w.t, 0, 0, 1, None, c0, c1)
            e1.record(stream)
            e1.synchronize()
            out.append(e0.elapsed_time(e1))
            if stats is not None:
                tm = dp.timing()
                stats["kern_ms"].append(tm.kernel_ms)
                stats["roll_ms"].append(tm.rollout_ms)
                stats["steps"] += tm.executed_steps
                stats["states"] += tm.checked_states
                stats["launches"] += tm.launches
                stats["refined"] += max(tm.refined, 0)
        return out

    c0, c1 = shard_range(model.n_candidates, rank, world)
    device_rounds(c0, c1, a.warmup)
    st = {"kern_ms": [], "roll_ms": [], "steps": 0, "states": 0, "launches": 0, "refined": 0}
    barrier()
    with ClockSampler(local) as clocks:
        dev_ms = device_rounds(c0, c1, a.steps, st)
        barrier()
        total_ms = max_over_ranks(sum(dev_ms))
        value = model.n_candidates * H * a.steps / (total_ms * 1e-3)

        # strong scaling: the BASELINE latency workload (2^20 candidates in
        # total) split over the ranks
        s0, s1 = shard_range(per_gpu, rank, world)
        device_rounds(s0, s1, a.warmup)
        barrier()
        strong_ms = max_over_ranks(sum(device_rounds(s0, s1, a.steps))) / a.steps
        barrier()

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
            if shared:  # ranks sharing a GPU: NCCL refuses; records over gloo
                sp = ShardedPlanner.on_shared_device(model, rank, world)
            else:
                sp = ShardedPlanner.on_device(model, rank, world)
                assert sp.exchange() == "nccl", sp.exchange()

            def e2e_step():
                return sp.plan_step(w.snapshot, w.t).action[0]

            def e2e_timing():
                return sp.device_planner.timing()

        for _ in range(a.warmup):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        h2d = d2h = 0
        e2e_each = []  # per call (median and best besides the mean)
        for _ in range(a.steps):
            tc = time.perf_counter()
            e2e_step()
            e2e_each.append(time.perf_counter() - tc)
            tm = e2e_timing()
            h2d += tm.h2d_bytes
            d2h += tm.d2h_bytes
        barrier()
        e2e_s = time.perf_counter() - t0
    e2e_s = max_over_ranks(e2e_s)
    e2e_median_ms = 1e3 * max_over_ranks(float(np.median(e2e_each)))
    e2e_best_ms = 1e3 * max_over_ranks(float(np.min(e2e_each)))
    e2e_value = model.n_candidates * H * a.steps / e2e_s

    # ---------------- roofline ------------------------------------------------
    round_avg_ms = sum(st["kern_ms"]) / len(st["kern_ms"])
    # the dominant kernel alone (the rollout, refill_kernel): its device span
    # from %globaltimer, first CTA start to last CTA end
    kern_avg_ms = sum(st["roll_ms"]) / len(st["roll_ms"])
    flops = workloads.algorithmic_flops([5, 2, 2], N, st["steps"] // a.steps,
                                        st["states"] // a.steps)
    achieved = flops / (kern_avg_ms * 1e-3) / 1e12
    traffic, traffic_live, pipes = None, None, None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        tj = json.loads(tf.read_text())
        traffic = tj.get("dram_bytes_per_launch")
        traffic_live = tj.get("live_dram_bytes_per_launch")
        pipes = tj.get("pipes")

    if rank == 0:
        cpu = None
        if world == 1:
            cpu = cpu_protocol(w.snapshot, w.t, H, model.n_candidates, a.cpu_seconds)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if a.precision == 32 else "f64", "data": "synthetic",
            "config": bench_config(a, world),
            "method": {"rollout_precision": "fp32" if a.precision == 32 else "fp64",
                       "winner": "certified: FP32 window re-ranked in the reference's FP64 "
                                 "arithmetic (PlannerConfig.refine)",
                       "l2": "flushed (256 MiB write) between timed steps",
                       **({"devices_shared": f"{world} ranks on {n_dev} GPU(s): code-path "
                                             "check only, not a scaling measurement"}
                          if shared else {})},
            "value_timing": "CUDA events on the planner stream around each sampling round "
                            "(generate + rollout + window-select kernels and the host "
                            "certification between them), snapshot resident in HBM, max over "
                            "ranks",
            "strong": {"samples_total": per_gpu, "ms_per_step": strong_ms,
                       "value": per_gpu * H / (strong_ms * 1e-3), "unit": UNIT},
            "near_tie_candidates_per_step": st["refined"] // a.steps,
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_s / a.steps * 1e3,
                    "ms_median": e2e_median_ms, "ms_best": e2e_best_ms,
                    "h2d_bytes_per_step": h2d // a.steps, "d2h_bytes_per_step": d2h // a.steps,
                    "api": "paraplan.Planner.plan_step" if world == 1 else
                           ("ShardedPlanner.plan_step on ranks sharing a GPU (winner records "
                            "exchanged over gloo; NCCL refuses a shared device)" if shared else
                            "pp_plan_step on a pp_comm_init rank (C++ sharded planner: "
                            "ncclAllReduce(min) of packed winner keys + ncclAllGather of "
                            "exact bests)")},
            "latency_ms": e2e_s / a.steps * 1e3,
            "gpu_launches": st["launches"],
            "nccl": ({"ranks": world, "version": ".".join(map(str, torch.cuda.nccl.version()))}
                     if world > 1 and not shared else None),
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": achieved / peak_tf if peak_tf else None,
                         "traffic": traffic, "traffic_live": traffic_live,
                         "peak_source": "FFMA loop measured in this run",
                         "ncu_pipes": pipes,
                         "kernel": "refill_kernel (rollout)", "kernel_ms": kern_avg_ms,
                         "kernel_timing": "%globaltimer span inside the kernel, averaged over "
                                          "the timed rounds",
                         "round_ms": round_avg_ms, "flops_per_launch": flops,
                         "executed_steps_per_launch": st["steps"] // a.steps},
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
    elif a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a))
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
