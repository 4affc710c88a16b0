"""ctypes mirror of the C-ABI PODs in include/paraplan_cuda.h.

Shared by the product loader (`capi.py`) and the test-side oracle loaders so a
test can hand byte-identical models and snapshots to the device planner, the
reference compiled from its sources, and the C restatement.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

PP_FP32 = 32
PP_FP64 = 64


class pp_vehicle(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "l_f", "l_r", "delta_max", "delta_rate_max", "u_v_min", "u_v_max",
        "overhang_front", "overhang_rear", "half_width", "T_s")]


class pp_norm(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("d_xi", "d_eta", "d_phi", "d_v")]


class pp_config(C.Structure):
    _fields_ = [
        ("H", C.c_int32), ("n_restarts", C.c_int32), ("n_iter_max", C.c_int32),
        ("n_candidates", C.c_int32), ("n_obst_pts", C.c_int32), ("early_exit", C.c_int32),
        ("eps_xi", C.c_double), ("eps_eta", C.c_double), ("eps_phi", C.c_double),
        ("eps_v", C.c_double), ("sigma_log_low", C.c_double), ("sigma_log_high", C.c_double),
        ("master_seed", C.c_uint64), ("threads", C.c_int32), ("precision", C.c_int32),
        ("device", C.c_int32), ("refine", C.c_int32), ("n_devices", C.c_int32),
        ("devices", C.c_int32 * 8),
    ]


class pp_model(C.Structure):
    _fields_ = [("vehicle", pp_vehicle), ("norm", pp_norm), ("config", pp_config),
                ("layer_sizes", C.POINTER(C.c_int32)), ("n_layers", C.c_int32)]


class pp_snapshot(C.Structure):
    _fields_ = [
        ("ev_x", C.c_double), ("ev_y", C.c_double), ("ev_phi", C.c_double), ("ev_v", C.c_double),
        ("actuator_delta", C.c_double), ("prev_a0", C.c_double), ("prev_a1", C.c_double),
        ("goal_x", C.c_double), ("goal_y", C.c_double), ("goal_phi", C.c_double),
        ("goal_v", C.c_double), ("field_xy", C.POINTER(C.c_double)), ("field_H", C.c_int32),
        ("n_points", C.c_int32), ("warm_theta", C.POINTER(C.c_double)),
        ("warm_theta_len", C.c_int32), ("_pad", C.c_int32),
    ]


class pp_snapshot_points(C.Structure):
    _fields_ = [
        ("ev_x", C.c_double), ("ev_y", C.c_double), ("ev_phi", C.c_double), ("ev_v", C.c_double),
        ("actuator_delta", C.c_double), ("prev_a0", C.c_double), ("prev_a1", C.c_double),
        ("goal_x", C.c_double), ("goal_y", C.c_double), ("goal_phi", C.c_double),
        ("goal_v", C.c_double), ("points", C.POINTER(C.c_double)), ("n_points", C.c_int32),
        ("_pad", C.c_int32), ("T_s", C.c_double), ("warm_theta", C.POINTER(C.c_double)),
        ("warm_theta_len", C.c_int32), ("_pad2", C.c_int32),
    ]


class pp_rollout_stats(C.Structure):
    _fields_ = [("reached", C.c_int32), ("t_goal", C.c_int32), ("collided", C.c_int32),
                ("steps", C.c_int32), ("path_length", C.c_double),
                ("terminal_cost", C.c_double), ("first_a0", C.c_double),
                ("first_a1", C.c_double)]


class pp_record(C.Structure):
    _fields_ = [("cls", C.c_int32), ("candidate", C.c_int32), ("restart", C.c_int32),
                ("iter", C.c_int32), ("k1", C.c_double), ("k2", C.c_double)]


class pp_plan_output(C.Structure):
    _fields_ = [("best_theta", C.POINTER(C.c_double)), ("trajectory", C.POINTER(C.c_double)),
                ("trajectory_len", C.c_int32), ("success", C.c_int32),
                ("action_a0", C.c_double), ("action_a1", C.c_double),
                ("predicted", pp_rollout_stats), ("evaluated", C.c_int64),
                ("winner", pp_record)]


class pp_timing(C.Structure):
    _fields_ = [("kernel_ms", C.c_double), ("executed_steps", C.c_int64),
                ("checked_states", C.c_int64), ("samples", C.c_int64),
                ("launches", C.c_int32), ("refined", C.c_int32),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("certify_ms", C.c_double), ("rollout_ms", C.c_double),
                ("fp64_rounds", C.c_int32), ("_pad", C.c_int32)]


# numpy view of pp_rollout_stats arrays (same layout, 48 bytes)
STATS_DTYPE = np.dtype([("reached", "<i4"), ("t_goal", "<i4"), ("collided", "<i4"),
                        ("steps", "<i4"), ("path_length", "<f8"), ("terminal_cost", "<f8"),
                        ("first_a0", "<f8"), ("first_a1", "<f8")])
assert STATS_DTYPE.itemsize == C.sizeof(pp_rollout_stats)
RECORD_DTYPE = np.dtype([("cls", "<i4"), ("candidate", "<i4"), ("restart", "<i4"),
                         ("iter", "<i4"), ("k1", "<f8"), ("k2", "<f8")])
assert RECORD_DTYPE.itemsize == C.sizeof(pp_record)


@dataclass
class Model:
    """Python-side bundle of the Planner constructor arguments, defaulted to
    the reference defaults (dynamics.hpp:9-27, policy.hpp:34-39,
    planner.hpp:14-35)."""

    layer_sizes: Sequence[int] = (5, 2, 2)
    H: int = 200
    n_restarts: int = 15
    n_iter_max: int = 1
    n_candidates: int = 20480
    n_obst_pts: int = 20
    early_exit: bool = False
    eps_xi: float = 1.0
    eps_eta: float = 0.25
    eps_phi: float = 10.0 * math.pi / 180.0
    eps_v: float = 5.0 / 3.6
    sigma_log_low: float = -2.0
    sigma_log_high: float = 1.0
    master_seed: int = 0
    threads: int = 1
    precision: int = PP_FP32
    device: int = 0
    refine: int = 1
    devices: Sequence[int] = ()  # several GPUs in one process (empty: `device`)
    vehicle: dict = field(default_factory=dict)
    norm: dict = field(default_factory=dict)

    def param_count(self) -> int:
        s = list(self.layer_sizes)
        return sum((s[i] + 1) * s[i + 1] for i in range(len(s) - 1))

    def to_c(self) -> pp_model:
        v = dict(l_f=1.1, l_r=1.4, delta_max=40.0 * math.pi / 180.0,
                 delta_rate_max=20.0 * math.pi / 180.0, u_v_min=-100.0 / (3.8 * 3.6),
                 u_v_max=100.0 / (7.4 * 3.6), overhang_front=0.7, overhang_rear=0.6,
                 half_width=1.0, T_s=0.1)
        v.update(self.vehicle)
        n = dict(d_xi=30.0, d_eta=3.5, d_phi=2.0 * math.pi, d_v=120.0 / 3.6)
        n.update(self.norm)
        m = pp_model()
        for k, val in v.items():
            setattr(m.vehicle, k, val)
        for k, val in n.items():
            setattr(m.norm, k, val)
        c = m.config
        for k in ("H", "n_restarts", "n_iter_max", "n_candidates", "n_obst_pts", "eps_xi",
                  "eps_eta", "eps_phi", "eps_v", "sigma_log_low", "sigma_log_high",
                  "master_seed", "threads", "precision", "device", "refine"):
            setattr(c, k, getattr(self, k))
        c.early_exit = int(bool(self.early_exit))
        if len(self.devices) > 8:
            raise ValueError("at most 8 devices per planner")
        c.n_devices = len(self.devices)
        for k, d in enumerate(self.devices):
            c.devices[k] = d
        arr = (C.c_int32 * len(self.layer_sizes))(*self.layer_sizes)
        m.layer_sizes = arr
        m.n_layers = len(self.layer_sizes)
        m._keep = arr  # keep the array alive with the struct
        return m


@dataclass
class Snapshot:
    """PlanningSnapshot (planner.hpp:39-46); field is (H+1, N, 2) float64."""

    ev: tuple = (0.0, 0.0, 0.0, 0.0)
    actuator_delta: float = 0.0
    prev_action: tuple = (0.0, 0.0)
    goal: tuple = (0.0, 0.0, 0.0, 0.0)
    field: np.ndarray | None = None
    warm_theta: np.ndarray | None = None

    def field_array(self, H: int) -> np.ndarray:
        if self.field is None:
            return np.zeros((H + 1, 0, 2), dtype=np.float64)
        return np.ascontiguousarray(self.field, dtype=np.float64)

    def to_c(self, H: int) -> pp_snapshot:
        s = pp_snapshot()
        s.ev_x, s.ev_y, s.ev_phi, s.ev_v = map(float, self.ev)
        s.actuator_delta = float(self.actuator_delta)
        s.prev_a0, s.prev_a1 = map(float, self.prev_action)
        s.goal_x, s.goal_y, s.goal_phi, s.goal_v = map(float, self.goal)
        f = self.field_array(H)
        s.field_H = f.shape[0] - 1
        s.n_points = f.shape[1]
        s.field_xy = f.ctypes.data_as(C.POINTER(C.c_double))
        keep = [f]
        if self.warm_theta is not None and len(self.warm_theta) > 0:
            w = np.ascontiguousarray(self.warm_theta, dtype=np.float64)
            s.warm_theta = w.ctypes.data_as(C.POINTER(C.c_double))
            s.warm_theta_len = len(w)
            keep.append(w)
        s._keep = keep
        return s


def points_snapshot(snap: Snapshot, points: np.ndarray, T_s: float = 0.1) -> pp_snapshot_points:
    """pp_snapshot_points of `snap` (its field ignored) with raw anchor-frame
    points (N, 4): x, y, heading, speed."""
    p = pp_snapshot_points()
    p.ev_x, p.ev_y, p.ev_phi, p.ev_v = map(float, snap.ev)
    p.actuator_delta = float(snap.actuator_delta)
    p.prev_a0, p.prev_a1 = map(float, snap.prev_action)
    p.goal_x, p.goal_y, p.goal_phi, p.goal_v = map(float, snap.goal)
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 4))
    p.points = pts.ctypes.data_as(C.POINTER(C.c_double))
    p.n_points = len(pts)
    p.T_s = T_s
    keep = [pts]
    if snap.warm_theta is not None and len(snap.warm_theta) > 0:
        w = np.ascontiguousarray(snap.warm_theta, dtype=np.float64)
        p.warm_theta = w.ctypes.data_as(C.POINTER(C.c_double))
        p.warm_theta_len = len(w)
        keep.append(w)
    p._keep = keep
    return p


def extrapolate(points: np.ndarray, H: int, T_s: float = 0.1) -> np.ndarray:
    """Constant-velocity field (geometry.cpp:43-61) from (N, 4) points
    (x, y, heading, speed) already in the anchor frame; expression order as the
    reference (step computed once per point, then x + h * step)."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 4)
    out = np.zeros((H + 1, len(pts), 2), dtype=np.float64)
    for j, (x, y, hd, sp) in enumerate(pts):
        sx = T_s * sp * math.cos(hd)
        sy = T_s * sp * math.sin(hd)
        for h in range(H + 1):
            out[h, j, 0] = x + h * sx
            out[h, j, 1] = y + h * sy
    return out


def plan_output_buffers(n_params: int, H: int):
    theta = np.zeros(n_params, dtype=np.float64)
    traj = np.zeros((H + 1, 4), dtype=np.float64)
    o = pp_plan_output()
    o.best_theta = theta.ctypes.data_as(C.POINTER(C.c_double))
    o.trajectory = traj.ctypes.data_as(C.POINTER(C.c_double))
    return o, theta, traj


def stats_to_dict(s: pp_rollout_stats) -> dict:
    return {k: getattr(s, k) for k, _ in pp_rollout_stats._fields_}
