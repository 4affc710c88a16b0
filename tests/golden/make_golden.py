"""Generate the golden vectors under tests/golden/ from the REFERENCE itself.

Runs the unmodified reference planner compiled from /root/reference/proj/src
(oracle/_ref/libparaplan_ref.so, built by `make -C oracle`). Doubles are
stored as float.hex() strings so every value round-trips bit-exactly.
Run from the repo root:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref, build  # noqa: E402
from paper_1904_06680_b200 import abi  # noqa: E402

OUT = Path(__file__).resolve().parent


def hx(a):
    a = np.asarray(a, dtype=np.float64).ravel()
    return [float(x).hex() for x in a]


def stats_json(s):
    return {k: (s[k].item() if s.dtype[k].kind == "i" else float(s[k]).hex())
            for k in s.dtype.names}


def snap_json(s: abi.Snapshot):
    return {"ev": hx(s.ev), "actuator_delta": float(s.actuator_delta).hex(),
            "prev_action": hx(s.prev_action), "goal": hx(s.goal),
            "field_shape": list(s.field.shape) if s.field is not None else [0, 0, 2],
            "field": hx(s.field) if s.field is not None else [],
            "warm_theta": hx(s.warm_theta) if s.warm_theta is not None else []}


def snapshots():
    c1 = Ref.builtin_snapshot("exp3_explicit", 0, 20, drop_dynamic=True)
    e3 = Ref.builtin_snapshot("exp3_explicit", 0, 30)
    park = Ref.builtin_snapshot("exp5_3wp", 0, 40)
    degenerate = abi.Snapshot(ev=(0.0, 0.0, 0.0, 0.0), goal=(0.0, 0.0, 0.0, 0.0),
                              field=np.zeros((21, 0, 2)))
    turn = abi.Snapshot(ev=(1.0, -2.0, 0.3, 2.0), actuator_delta=0.1, prev_action=(0.2, -0.1),
                        goal=(8.0, 3.0, 1.2, 1.0), field=np.zeros((41, 0, 2)))
    return {"c1": (c1, 20), "exp3_explicit_t0": (e3, 30), "exp5_3wp_t0": (park, 40),
            "degenerate": (degenerate, 20), "turn": (turn, 40)}


def main():
    build()
    gold = {"source": "reference planner compiled from /root/reference/proj/src "
                      "(oracle/_ref/libparaplan_ref.so)"}
    # KeyedRng streams (src/rng.cpp:26-58)
    keys = [(1, 2, 3, 4, 5), (0, 0, 0, 0, 1), (42, 7, 3, 1, 99), (12345, 7, 14, 0, 20479)]
    gold["rng"] = [{"key": list(k),
                    "u64": [format(int(x), "016x") for x in Ref.rng_stream(k, 0, 8)],
                    "unit": hx(Ref.rng_stream(k, 1, 8)),
                    "normal": hx(Ref.rng_stream(k, 2, 9))} for k in keys]
    # sample_candidate (src/planner.cpp:207-226)
    cands = []
    for sizes in ([5, 2, 2], [5, 10, 2]):
        m = abi.Model(layer_sizes=sizes, master_seed=12345)
        r = Ref(m)
        center = np.linspace(-0.5, 0.5, m.param_count())
        for (t, rs, it, c) in [(0, 0, 0, 0), (0, 0, 0, 1), (7, 3, 0, 2), (7, 14, 1, 999)]:
            cands.append({"sizes": sizes, "seed": 12345, "t": t, "restart": rs, "iter": it,
                          "cand": c, "center": hx(center),
                          "theta": hx(r.sample_candidate(center, t, rs, it, c)),
                          "sigma": float(r.perturbation_sigma(t, rs, it, c)).hex()})
    gold["sample_candidate"] = cands

    snaps = snapshots()
    gold["snapshots"] = {k: {"H": H, **snap_json(s)} for k, (s, H) in snaps.items()}

    # per-candidate stats of one sampling round (evaluate_block's per-sample work)
    rounds = []
    for key, n in (("c1", 256), ("exp3_explicit_t0", 256), ("exp5_3wp_t0", 128), ("turn", 128)):
        s, H = snaps[key]
        m = abi.Model(H=H, n_restarts=1, n_candidates=n, master_seed=3)
        r = Ref(m)
        st = r.eval_candidates(s, 5, 0, 0, np.zeros(m.param_count()), 0, n)
        rounds.append({"snapshot": key, "H": H, "seed": 3, "t": 5, "n": n,
                       "stats": [stats_json(x) for x in st]})
    gold["rounds"] = rounds

    # full plan_step outputs (src/planner.cpp:238-351)
    plans = []
    cases = [("c1", dict(n_restarts=1, n_candidates=512), 0),
             ("exp3_explicit_t0", dict(n_restarts=3, n_candidates=200, master_seed=9), 4),
             ("exp5_3wp_t0", dict(n_restarts=2, n_iter_max=2, n_candidates=96, master_seed=5), 1),
             ("degenerate", dict(n_restarts=2, n_candidates=24), 0),
             ("degenerate", dict(n_restarts=6, n_candidates=16, early_exit=True), 0),
             ("turn", dict(n_restarts=4, n_iter_max=2, n_candidates=32, master_seed=17), 2)]
    for key, kw, t in cases:
        s, H = snaps[key]
        m = abi.Model(H=H, **kw)
        o, theta, traj = Ref(m).plan_step(s, t)
        plans.append({"snapshot": key, "H": H, "config": kw, "t": t,
                      "best_theta": hx(theta), "trajectory": hx(traj),
                      "action": hx([o.action_a0, o.action_a1]), "success": o.success,
                      "evaluated": o.evaluated,
                      "predicted": {"reached": o.predicted.reached, "t_goal": o.predicted.t_goal,
                                    "collided": o.predicted.collided,
                                    "path_length": float(o.predicted.path_length).hex(),
                                    "terminal_cost": float(o.predicted.terminal_cost).hex()}})
    gold["plans"] = plans
    (OUT / "reference_vectors.json").write_text(json.dumps(gold, indent=1))
    print("wrote", OUT / "reference_vectors.json")


if __name__ == "__main__":
    main()
