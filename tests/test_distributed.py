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


# ---- the packed-key winner collective (csrc/cuda/keypack.h) -------------

def _ref_order_key(cls, t_goal, cost, idx):
    """The reference's order (better(), src/planner.cpp:40-44; ties to the
    lowest index) as a Python sort key: smaller is better."""
    return (-cls, t_goal if cls == 2 else 0, cost, idx)


def test_packed_key_order_is_the_reference_order():
    from paper_1904_06680_b200 import capi
    rng = np.random.default_rng(5)
    keys = []
    for _ in range(4000):
        cls = int(rng.integers(0, 3))
        tg = int(rng.integers(0, 256)) if cls == 2 else 0
        # float costs, with deliberate exact ties
        cost = float(np.float32(rng.choice([0.5, 1.25, rng.uniform(0, 50)])))
        idx = int(rng.integers(0, 1 << 22))
        keys.append((cls, tg, cost, idx))
    packed = [capi.pack_key(*k) for k in keys]
    by_pack = [keys[i] for i in np.argsort(np.array(packed, dtype=np.uint64), kind="stable")]
    by_ref = sorted(keys, key=lambda k: _ref_order_key(*k))
    assert by_pack == by_ref
    for k, p in zip(keys, packed):
        assert capi.unpack_key(p) == k
    assert capi.pack_key(-1, 0, 0.0, 0) == (1 << 64) - 1


def _key_worker(rank, world, port_no, results):
    """Each rank evaluates its contiguous shard with the oracle, packs its
    best, and the ranks min-reduce over gloo: the reduced key must be the
    single-process winner (the C++ planner does the same with ncclMin)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from paper_1904_06680_b200 import capi
    for name, t_snap, cfg, t in CASES:
        model = abi.Model(**cfg)
        snap = Ref.builtin_snapshot(name, t_snap, model.H)
        port = Port(model)
        n = model.n_candidates
        c0, c1 = shard_range(n, rank, world)
        st = port.eval_candidates(snap, t, 0, 0, np.zeros(model.param_count()), c0, c1)
        best = (1 << 64) - 1
        for i, s in enumerate(st):
            cls = 0 if s["collided"] else (2 if s["reached"] else 1)
            cost = s["path_length"] if cls == 2 else s["terminal_cost"]
            best = min(best, capi.pack_key(cls, int(s["t_goal"]), float(np.float32(cost)), c0 + i))
        # gloo reduces int64: flip the sign bit so the signed order is the
        # unsigned one
        x = torch.tensor([best ^ (1 << 63)], dtype=torch.uint64).view(torch.int64)
        dist.all_reduce(x, op=dist.ReduceOp.MIN)
        results[(rank, name)] = int(x.view(torch.uint64).item()) ^ (1 << 63)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_packed_winner_allreduce_over_ranks(world):
    from paper_1904_06680_b200 import capi
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.spawn(_key_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for name, t_snap, cfg, t in CASES:
        model = abi.Model(**cfg)
        snap = Ref.builtin_snapshot(name, t_snap, model.H)
        st = Port(model).eval_candidates(snap, t, 0, 0, np.zeros(model.param_count()), 0,
                                         model.n_candidates)
        keys = []
        for i, s in enumerate(st):
            cls = 0 if s["collided"] else (2 if s["reached"] else 1)
            cost = s["path_length"] if cls == 2 else s["terminal_cost"]
            keys.append(capi.pack_key(cls, int(s["t_goal"]), float(np.float32(cost)), i))
        want = min(keys)
        for rank in range(world):
            assert results[(rank, name)] == want, (name, rank)
