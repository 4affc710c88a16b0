"""Multi-rank plan_step (paper_1904_06680_b200.distributed) on CPU:
world_size 2 and 3 over gloo, the device round replaced by the C restatement
evaluating each rank's candidate shard. The merged plan must be bit-identical
to the single-process reference schedule (planner_test.cpp:209-241 analogue
across ranks instead of threads)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Port, Ref
from paper_1904_06680_b200 import abi
from paper_1904_06680_b200.distributed import ShardedPlanner, merge_ordered, shard_range

CASES = [
    ("exp3_explicit", 0, dict(H=30, n_restarts=3, n_candidates=101, master_seed=9), 4),
    ("exp5_3wp", 0, dict(H=40, n_restarts=2, n_iter_max=2, n_candidates=64, master_seed=5), 1),
    ("exp1", 0, dict(H=40, n_restarts=4, n_candidates=50, early_exit=True), 0),
]


def port_evaluate(model):
    port = Port(model)

    def evaluate(snap, t, it, r0, rc, center, c0, c1):
        out = np.zeros(rc, dtype=abi.RECORD_DTYPE)
        for k in range(rc):
            st = port.eval_candidates(snap, t, it, r0 + k, center, c0, c1)
            best = None
            for i, s in enumerate(st):
                cls = 0 if s["collided"] else (2 if s["reached"] else 1)
                k1 = -float(s["t_goal"]) if cls == 2 else -s["terminal_cost"]
                k2 = -s["path_length"] if cls == 2 else 0.0
                rec = (cls, c0 + i, r0 + k, it, k1, k2)
                best = merge_ordered([best, rec] if best else [rec])
            out[k] = best if best else (-1, -1, r0 + k, it, 0.0, 0.0)
        return out

    return evaluate, port


def _worker(rank, world, port_no, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    def all_gather(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)
        return torch.stack(outs).numpy()

    for name, t_snap, cfg, t in CASES:
        model = abi.Model(**cfg)
        snap = Ref.builtin_snapshot(name, t_snap, model.H)
        evaluate, port = port_evaluate(model)
        sp = ShardedPlanner(model, rank, world, evaluate, port, all_gather)
        r = sp.plan_step(snap, t)
        results[(rank, name)] = (r.best_theta.tobytes(), r.trajectory.tobytes(), r.action,
                                 r.evaluated, r.success)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_plan_matches_single_process(world):
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for name, t_snap, cfg, t in CASES:
        model = abi.Model(**cfg)
        snap = Ref.builtin_snapshot(name, t_snap, model.H)
        o, theta, traj = Port(model).plan_step(snap, t)
        for rank in range(world):
            bt, tr, action, evaluated, success = results[(rank, name)]
            assert bt == theta.tobytes(), (name, rank)
            assert tr == traj.tobytes()
            assert action == (o.action_a0, o.action_a1)
            assert evaluated == o.evaluated and success == bool(o.success)


def test_shard_ranges_partition_in_order():
    for n in (1, 7, 1 << 20):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
