"""The multi-GPU plan_step on real device rounds: two ranks (gloo for the
record exchange) each run the sm_100a kernels on their candidate shard of the
same GPU -- no kernel waits on another rank, the ranks only exchange winner
records on the host -- and must return the single-GPU plan bit for bit."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1904_06680_b200 import abi, capi, workloads

pytestmark = pytest.mark.gpu

CFGS = [dict(H=30, n_restarts=1, n_candidates=1 << 16),
        dict(H=30, n_restarts=3, n_candidates=5000, master_seed=4),
        dict(H=30, n_restarts=2, n_iter_max=2, n_candidates=3000, master_seed=8)]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1904_06680_b200.distributed import ShardedPlanner
    w = workloads.c2(samples=1 << 10)
    for k, cfg in enumerate(CFGS):
        sp = ShardedPlanner.on_shared_device(abi.Model(**cfg), rank, world)
        r = sp.plan_step(w.snapshot, w.t)
        out[(rank, k)] = (r.best_theta.tobytes(), r.trajectory.tobytes(), r.action, r.evaluated,
                          r.winner[:2])
        sp.device_planner.close()
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_equal_one_gpu_plan():
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
    w = workloads.c2(samples=1 << 10)
    for k, cfg in enumerate(CFGS):
        o, theta, traj = capi.DevicePlanner(abi.Model(**cfg)).plan_step(w.snapshot, w.t)
        for rank in range(2):
            bt, tr, action, evaluated, win = out[(rank, k)]
            assert bt == theta.tobytes() and tr == traj.tobytes(), (k, rank)
            assert action == (o.action_a0, o.action_a1) and evaluated == o.evaluated


@pytest.mark.parametrize("cfg", CFGS + [dict(H=30, n_restarts=15, n_candidates=20480)])
@pytest.mark.parametrize("shards", [2, 3])
def test_in_process_shards_equal_one_gpu_plan(cfg, shards):
    """PlannerConfig.devices: one process drives several shards (here all on
    cuda:0, each with its own stream and certification pool); the plan is
    the single-shard plan bit for bit, for the field and the raw-points path."""
    w = workloads.c2(samples=1 << 10)
    one = capi.DevicePlanner(abi.Model(**cfg))
    many = capi.DevicePlanner(abi.Model(**cfg, devices=[0] * shards))
    o1, th1, tr1 = one.plan_step(w.snapshot, w.t)
    o2, th2, tr2 = many.plan_step(w.snapshot, w.t)
    assert np.array_equal(th1, th2) and np.array_equal(tr1, tr2)
    assert (o1.action_a0, o1.action_a1, o1.evaluated, o1.success) == \
        (o2.action_a0, o2.action_a1, o2.evaluated, o2.success)
    assert (o1.winner.restart, o1.winner.candidate) == (o2.winner.restart, o2.winner.candidate)
    t = many.timing()
    assert t.launches >= 3 * shards and t.samples >= o1.evaluated
    many.close()
    one.close()


def test_in_process_shards_closed_loop_matches_one_gpu():
    """run_mission through the drop-in module with PlannerConfig.devices."""
    from paper_1904_06680_b200 import import_paraplan
    pp = import_paraplan()
    logs = []
    for devices in ([], [0, 0]):
        spec = pp.builtin_scenario("exp3_explicit")
        c = spec.planner
        c.H, c.n_restarts, c.n_candidates = 30, 2, 4096
        c.devices = devices
        spec.mission.time_limit = 1.0
        logs.append(pp.run_mission(spec.mission, c, spec.arch, 0))
    a, b = logs
    assert len(a.records) == len(b.records) > 0
    for ra, rb in zip(a.records, b.records):
        assert (ra.state.x, ra.state.y, ra.state.phi, ra.state.v) == \
            (rb.state.x, rb.state.y, rb.state.phi, rb.state.v)


def test_in_process_shards_reject_a_missing_device():
    import torch
    bad = torch.cuda.device_count()  # one past the last ordinal
    with pytest.raises(ValueError, match="out of range"):
        capi.DevicePlanner(abi.Model(H=30, n_restarts=1, n_candidates=1024, devices=[0, bad]))
    # the failed construction left no shard behind: a good planner still works
    w = workloads.c2(samples=1 << 10)
    dp = capi.DevicePlanner(abi.Model(H=30, n_restarts=1, n_candidates=1024, devices=[0, 0]))
    o, _, _ = dp.plan_step(w.snapshot, w.t)
    assert o.evaluated == 1024


@pytest.mark.parametrize("cfg", CFGS + [dict(H=30, n_restarts=15, n_candidates=20480),
                                        dict(H=200, n_restarts=1, n_candidates=1 << 15)])
def test_one_rank_nccl_communicator_equals_unsharded(cfg):
    """pp_comm_init on a one-rank NCCL communicator runs the whole sharded
    path on one GPU: packed winner keys, the in-stream
    ncclAllReduce(ncclMin, uint64), the globally anchored window, the
    ncclAllGather of exact bests -- and returns the unsharded plan."""
    w = workloads.c2(samples=1 << 10)
    m = workloads.c2_mission()
    snap = w.snapshot if cfg["H"] == 30 else workloads.snapshot_from_mission(
        m, m.initial_state, workloads.C2_T, cfg["H"], 20)
    one = capi.DevicePlanner(abi.Model(**cfg))
    comm = capi.DevicePlanner(abi.Model(**cfg))
    comm.join_communicator(capi.comm_unique_id(), 1, 0)
    assert comm.exchange() == "nccl" and one.exchange() == "none"
    o1, th1, tr1 = one.plan_step(snap, w.t)
    o2, th2, tr2 = comm.plan_step(snap, w.t)
    assert np.array_equal(th1, th2) and np.array_equal(tr1, tr2)
    assert (o1.winner.restart, o1.winner.candidate, o1.evaluated) == \
        (o2.winner.restart, o2.winner.candidate, o2.evaluated)
    # + the pack kernel and the NCCL kernel per round
    assert comm.timing().launches > one.timing().launches
    comm.close()
    one.close()


def test_in_process_shards_use_host_exchange_on_one_gpu():
    many = capi.DevicePlanner(abi.Model(H=30, n_restarts=1, n_candidates=4096, devices=[0, 0]))
    assert many.exchange() == "host"
    many.close()


def test_sharded_state0_stop_returns_candidate_zero():
    """Every rollout stops at state 0 (obstacle in the chassis): each shard
    certifies directly, and the winner is global candidate 0 (shard 0)."""
    field = np.zeros((31, 1, 2))
    snap = abi.Snapshot(ev=(0.0, 0.0, 0.0, 5.0), actuator_delta=0.2,
                        prev_action=(0.0, 0.32142857142857145), goal=(20.0, 0.0, 0.0, 5.0),
                        field=field)
    cfg = dict(H=30, n_restarts=2, n_candidates=6000)
    one = capi.DevicePlanner(abi.Model(**cfg))
    many = capi.DevicePlanner(abi.Model(**cfg, devices=[0, 0, 0]))
    o1, th1, _ = one.plan_step(snap, 0)
    o2, th2, _ = many.plan_step(snap, 0)
    assert o1.winner.candidate == o2.winner.candidate == 0
    assert np.array_equal(th1, th2) and o2.action_a1 == -1.0
