"""Multi-GPU plan_step: one process per GPU, candidates sharded.

The flat candidate index space of every restart is split into contiguous,
increasing ranges, rank r owning [n*r/W, n*(r+1)/W)
(/root/reference/proj/src/planner.cpp:280-281 splits worker ranges the same
way).

GPU ranks (`CommPlanner`): the planner itself is sharded in C++
(pp_comm_init, csrc/capi/round.cpp + exchange.cpp). Each rank's round runs on
its own GPU; one ncclAllReduce(ncclMin, uint64) of packed (class, t_goal,
FP32 cost, index) keys in the stream anchors every rank's near-tie window on
the global winner, the ranks certify their own window members in the
reference's FP64 arithmetic and all-gather the exact per-restart bests, so
every rank returns the same plan: the reference's ordered merge
(src/planner.cpp:310-321). Python only shares the NCCL unique id.

`ShardedPlanner` is the same partition and merge written in Python over any
per-shard evaluator and any all-gather: the CPU tests run it over gloo with
the C oracle as the shard evaluator (tests/test_distributed.py), and it
checks the packed-key reduction against the ordered merge.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import abi


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def key_better(a, b) -> bool:
    """better(ScoreKey, ScoreKey), src/planner.cpp:40-44."""
    if a[0] != b[0]:
        return a[0] > b[0]
    if a[1] != b[1]:
        return a[1] > b[1]
    return a[2] > b[2]


def merge_ordered(recs) -> tuple | None:
    """Strict-better scan over records in increasing index order; records
    are (cls, candidate, restart, iter, k1, k2); candidate < 0 = empty."""
    best = None
    for r in recs:
        if r[1] < 0:
            continue
        if best is None or key_better((r[0], r[4], r[5]), (best[0], best[4], best[5])):
            best = tuple(r)
    return best


@dataclass
class PlanResult:
    best_theta: np.ndarray
    action: tuple
    predicted: abi.pp_rollout_stats
    trajectory: np.ndarray
    success: bool
    evaluated: int
    winner: tuple


class ShardedPlanner:
    """plan_step over `world` ranks.

    evaluate(snap, t, it, r0, rc, center, c0, c1) -> record array (RECORD_DTYPE)
        the device round on this rank's shard (DevicePlanner.evaluate).
    host: object with sample_candidate(center, t, r, it, c) and
        rollout(snap, theta) -> (stats, traj) -- the FP64 host path.
    all_gather(np.ndarray (k, 6) float64) -> np.ndarray (world, k, 6)
    """

    def __init__(self, model: abi.Model, rank: int, world: int, evaluate, host, all_gather):
        self.model = model
        self.rank = rank
        self.world = world
        self._evaluate = evaluate
        self._host = host
        self._all_gather = all_gather
        self.n_params = model.param_count()

    @classmethod
    def on_device(cls, model: abi.Model, rank: int, world: int, group=None):
        """GPU ranks, one GPU each: the C++ sharded planner over NCCL."""
        return CommPlanner(model, rank, world, group)

    @classmethod
    def on_shared_device(cls, model: abi.Model, rank: int, world: int, group=None):
        """Ranks that share a GPU (NCCL refuses duplicate devices; a 1-GPU
        box): each rank's shard runs on the device through pp_evaluate and
        the winner records are all-gathered over the group's backend."""
        import torch
        import torch.distributed as dist

        from .capi import DevicePlanner

        dp = DevicePlanner(model)
        last = {"snap": None}

        def evaluate(snap, t, it, r0, rc, center, c0, c1):
            # upload the snapshot once per plan step (its first round is
            # iteration 0 of every restart); later rounds reuse it in HBM
            fresh = (it == 0 and r0 == 0) or snap is not last["snap"]
            last["snap"] = snap
            return dp.evaluate(snap if fresh else None, t, it, r0, rc, center, c0, c1)[0]

        dev = torch.device("cuda", model.device) if dist.get_backend(group) == "nccl" else "cpu"

        def all_gather(x: np.ndarray) -> np.ndarray:
            t = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
            if dev == "cpu":
                outs = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(outs, t, group=group)
                return torch.stack(outs).numpy()
            out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=dev)
            dist.all_gather_into_tensor(out, t, group=group)
            return out.cpu().numpy()

        sp = cls(model, rank, world, evaluate, dp, all_gather)
        sp.device_planner = dp
        return sp

    def _round(self, snap, t, it, r0, rc, center) -> list:
        c0, c1 = shard_range(self.model.n_candidates, self.rank, self.world)
        recs = self._evaluate(snap, t, it, r0, rc, center, c0, c1)
        local = np.array([[r["cls"], r["candidate"], r["restart"], r["iter"], r["k1"], r["k2"]]
                          for r in recs], dtype=np.float64).reshape(rc, 6)
        allr = self._all_gather(local)  # (world, rc, 6)
        merged = []
        for k in range(rc):
            m = merge_ordered([tuple(allr[w, k]) for w in range(self.world)])
            if m is None:
                m = (-1.0, -1.0, float(r0 + k), float(it), 0.0, 0.0)
            merged.append((int(m[0]), int(m[1]), int(m[2]), int(m[3]), m[4], m[5]))
        return merged

    def plan_step(self, snap: abi.Snapshot, t: int) -> PlanResult:
        m = self.model
        P = self.n_params
        if snap.warm_theta is not None and len(snap.warm_theta) not in (0, P):
            raise ValueError("warm start vector size mismatch")
        init = (np.asarray(snap.warm_theta, dtype=np.float64)
                if snap.warm_theta is not None and len(snap.warm_theta) == P else np.zeros(P))
        R, I, n = m.n_restarts, m.n_iter_max, m.n_candidates
        first = self._round(snap, t, 0, 0, R, init)  # iteration 0 of every restart
        best = None
        best_theta = np.zeros(P)
        any_free = False
        evaluated = 0
        done = False
        for r in range(R):
            for it in range(I):
                if it == 0:
                    center = init
                    rec = first[r]
                else:
                    center = best_theta if best is not None else center
                    rec = self._round(snap, t, it, r, 1, center)[0]
                evaluated += n
                any_free = any_free or rec[0] >= 1
                if best is None or key_better((rec[0], rec[4], rec[5]),
                                              (best[0], best[4], best[5])):
                    best_theta = self._host.sample_candidate(center, t, r, it, rec[1])
                    best = rec
                if m.early_exit and best is not None and best[0] == 2:
                    done = True
                    break
            if done:
                break
        st, traj = self._host.rollout(snap, best_theta)
        success = bool(st.reached) and not bool(st.collided)
        if any_free:
            action = (st.first_a0, st.first_a1)
        else:
            action = (snap.actuator_delta / m.to_c().vehicle.delta_max, -1.0)
        return PlanResult(best_theta, action, st, traj, success, evaluated, best)


class CommPlanner:
    """One rank of a sharded planner: a DevicePlanner joined to a `world`-rank
    NCCL communicator (the unique id travels over torch.distributed). Every
    rank calls plan_step with the same snapshot and gets the same plan."""

    def __init__(self, model: abi.Model, rank: int, world: int, group=None):
        import torch.distributed as dist

        from .capi import DevicePlanner, comm_unique_id

        self.model = model
        self.rank, self.world = rank, world
        self.device_planner = DevicePlanner(model)
        uid = [comm_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0, group=group)
        self.device_planner.join_communicator(uid[0], world, rank)

    def plan_step(self, snap: abi.Snapshot, t: int) -> PlanResult:
        o, theta, traj = self.device_planner.plan_step(snap, t)
        w = o.winner
        return PlanResult(theta, (o.action_a0, o.action_a1), o.predicted, traj, bool(o.success),
                          o.evaluated, (w.cls, w.candidate, w.restart, w.iter, w.k1, w.k2))

    def exchange(self) -> str:
        return self.device_planner.exchange()
