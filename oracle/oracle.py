"""TEST INFRASTRUCTURE: ctypes loaders for the two CPU checkers.

* `Ref`    -- oracle/_ref/libparaplan_ref.so, the unmodified reference planner
             compiled from /root/reference/proj/src by oracle/Makefile.
* `Port`   -- oracle/_ref/liboracle.so, the plain-C restatement
             (oracle/paraplan_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module. Both libraries are prebuilt here and travel to the GPU box; the
box never reads /root/reference.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_1904_06680_b200 import abi

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libparaplan_ref.so"
PORT_SO = HERE / "_ref" / "liboracle.so"
REF_SRC = Path("/root/reference/proj")


def build(quiet: bool = True) -> None:
    """Compile the checkers (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", str(HERE), f"-j{os.cpu_count() or 4}"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct))


class _Base:
    def _stats_array(self, n):
        return np.zeros(n, dtype=abi.STATS_DTYPE)


class Ref(_Base):
    """The reference Planner (C++ from /root/reference) behind ref_driver.cpp."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not REF_SO.exists():
                raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle`")
            L = C.CDLL(str(REF_SO))
            L.ref_create.restype = C.c_void_p
            L.ref_create.argtypes = [C.POINTER(abi.pp_model)]
            L.ref_destroy.argtypes = [C.c_void_p]
            L.ref_last_error.restype = C.c_char_p
            L.ref_param_count.argtypes = [C.c_void_p]
            L.ref_plan_step.argtypes = [C.c_void_p, C.POINTER(abi.pp_snapshot), C.c_uint64,
                                        C.POINTER(abi.pp_plan_output)]
            L.ref_rollout.argtypes = [C.c_void_p, C.POINTER(abi.pp_snapshot),
                                      C.POINTER(C.c_double), C.c_int32,
                                      C.POINTER(abi.pp_rollout_stats), C.POINTER(C.c_double),
                                      C.c_int32, C.POINTER(C.c_int32)]
            L.ref_sample_candidate.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int32,
                                               C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
                                               C.POINTER(C.c_double)]
            L.ref_perturbation_sigma.restype = C.c_double
            L.ref_perturbation_sigma.argtypes = [C.c_void_p, C.c_uint64, C.c_int32,
                                                 C.c_int32, C.c_int32]
            L.ref_eval_candidates.argtypes = [C.c_void_p, C.POINTER(abi.pp_snapshot),
                                              C.c_uint64, C.c_int32, C.c_int32,
                                              C.POINTER(C.c_double), C.c_int64, C.c_int64,
                                              C.c_void_p]
            L.ref_eval_theta.argtypes = [C.c_void_p, C.POINTER(abi.pp_snapshot),
                                         C.POINTER(C.c_double), C.c_int64, C.c_void_p]
            L.ref_rng_stream.argtypes = [C.c_uint64] * 5 + [C.c_int32, C.c_int32, C.c_void_p]
            L.ref_selfchecks.argtypes = [C.c_char_p, C.c_int32]
            L.ref_builtin_snapshot.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32,
                                               C.c_int32, C.POINTER(abi.pp_snapshot),
                                               C.POINTER(C.c_double), C.c_int64]
            L.ref_mission_snapshot.argtypes = [C.POINTER(C.c_double), C.c_int32,
                                               C.POINTER(C.c_double), C.c_int32,
                                               C.POINTER(C.c_double), C.c_int32,
                                               C.POINTER(C.c_double), C.c_int32, C.c_int32,
                                               C.c_int32, C.POINTER(abi.pp_snapshot),
                                               C.POINTER(C.c_double), C.c_int64]
            L.ref_spin_calibration.restype = C.c_double
            L.ref_spin_calibration.argtypes = [C.c_int32, C.c_double, C.c_int32]
            L.ref_acceptance9_snapshot.argtypes = [C.c_int32, C.c_int32,
                                                   C.POINTER(abi.pp_snapshot),
                                                   C.POINTER(C.c_double), C.c_int64,
                                                   C.POINTER(C.c_double),
                                                   C.POINTER(C.c_int32)]
            L.ref_run_mission_builtin.argtypes = [C.c_char_p, C.c_int32, C.c_int32,
                                                  C.c_int32, C.c_double, C.c_uint64,
                                                  C.c_int32, C.POINTER(C.c_double), C.c_int32,
                                                  C.POINTER(C.c_double)]
            L.ref_run_sweep_builtin.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32,
                                                C.c_double, C.POINTER(C.c_uint64), C.c_int32,
                                                C.c_int32, C.c_char_p]
            L.ref_serialize_builtin.argtypes = [C.c_char_p, C.c_char_p, C.c_int32]
            cls._lib = L
        return cls._lib

    def __init__(self, model: abi.Model):
        self.model = model
        self._m = model.to_c()
        self.h = self.lib().ref_create(C.byref(self._m))
        if not self.h:
            raise ValueError(self.lib().ref_last_error().decode())
        self.n_params = self.lib().ref_param_count(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib().ref_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc != 0:
            msg = self.lib().ref_last_error().decode()
            raise ValueError(msg) if rc == 1 else RuntimeError(msg)

    def plan_step(self, snap: abi.Snapshot, t: int):
        s = snap.to_c(self.model.H)
        o, theta, traj = abi.plan_output_buffers(self.n_params, self.model.H)
        self._check(self.lib().ref_plan_step(self.h, C.byref(s), t, C.byref(o)))
        return o, theta, traj[: o.trajectory_len].copy()

    def rollout(self, snap: abi.Snapshot, theta):
        s = snap.to_c(self.model.H)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        st = abi.pp_rollout_stats()
        traj = np.zeros((self.model.H + 1, 4))
        n = C.c_int32()
        self._check(self.lib().ref_rollout(self.h, C.byref(s), _ptr(th), len(th), C.byref(st),
                                           _ptr(traj), self.model.H + 1, C.byref(n)))
        return st, traj[: n.value].copy()

    def sample_candidate(self, center, t, restart, it, cand):
        c = np.ascontiguousarray(center, dtype=np.float64)
        out = np.zeros_like(c)
        self._check(self.lib().ref_sample_candidate(self.h, _ptr(c), len(c), t, restart, it,
                                                    cand, _ptr(out)))
        return out

    def perturbation_sigma(self, t, restart, it, cand):
        return self.lib().ref_perturbation_sigma(self.h, t, restart, it, cand)

    def eval_candidates(self, snap, t, it, restart, center, c_begin, c_end):
        s = snap.to_c(self.model.H)
        c = np.ascontiguousarray(center, dtype=np.float64)
        out = self._stats_array(c_end - c_begin)
        self._check(self.lib().ref_eval_candidates(self.h, C.byref(s), t, it, restart, _ptr(c),
                                                   c_begin, c_end, out.ctypes.data))
        return out

    def eval_theta(self, snap, theta):
        s = snap.to_c(self.model.H)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        out = self._stats_array(th.shape[0])
        self._check(self.lib().ref_eval_theta(self.h, C.byref(s), _ptr(th), th.shape[0],
                                              out.ctypes.data))
        return out

    @classmethod
    def rng_stream(cls, key, kind, n):
        out = np.zeros(n, dtype=np.uint64 if kind == 0 else np.float64)
        cls.lib().ref_rng_stream(*key, kind, n, out.ctypes.data)
        return out

    @classmethod
    def selfchecks(cls):
        buf = C.create_string_buffer(1 << 16)
        failed = cls.lib().ref_selfchecks(buf, len(buf))
        return failed, buf.value.decode()

    @classmethod
    def builtin_snapshot(cls, name, t, H, n_obst_pts=20, drop_dynamic=False):
        cap = 2 * (H + 1) * 4096
        field = np.zeros(cap)
        s = abi.pp_snapshot()
        n = cls.lib().ref_builtin_snapshot(name.encode(), t, H, n_obst_pts, int(drop_dynamic),
                                           C.byref(s), _ptr(field), cap)
        if n < 0:
            raise RuntimeError(cls.lib().ref_last_error().decode())
        return abi.Snapshot(ev=(s.ev_x, s.ev_y, s.ev_phi, s.ev_v),
                            actuator_delta=s.actuator_delta, prev_action=(s.prev_a0, s.prev_a1),
                            goal=(s.goal_x, s.goal_y, s.goal_phi, s.goal_v),
                            field=field[: 2 * (H + 1) * n].reshape(H + 1, n, 2).copy())


    @classmethod
    def mission_snapshot(cls, waypoints, static_pts, dyn_pts, ev, t, H, n_obst_pts):
        """Tick-t snapshot of a mission through the reference's own
        select_goal -> sense -> extrapolate (src/mission.cpp:124-144)."""
        wp = np.ascontiguousarray(waypoints, dtype=np.float64).reshape(-1, 4)
        st = np.ascontiguousarray(static_pts, dtype=np.float64).reshape(-1, 4)
        dy = np.ascontiguousarray(dyn_pts, dtype=np.float64).reshape(-1, 4)
        e = np.ascontiguousarray(ev, dtype=np.float64)
        cap = 2 * (H + 1) * max(n_obst_pts, 1)
        field = np.zeros(cap)
        s = abi.pp_snapshot()
        n = cls.lib().ref_mission_snapshot(_ptr(wp), len(wp), _ptr(st), len(st), _ptr(dy),
                                           len(dy), _ptr(e), t, H, n_obst_pts, C.byref(s),
                                           _ptr(field), cap)
        if n < 0:
            raise RuntimeError(cls.lib().ref_last_error().decode())
        return abi.Snapshot(ev=(s.ev_x, s.ev_y, s.ev_phi, s.ev_v),
                            actuator_delta=s.actuator_delta, prev_action=(s.prev_a0, s.prev_a1),
                            goal=(s.goal_x, s.goal_y, s.goal_phi, s.goal_v),
                            field=field[: 2 * (H + 1) * n].reshape(H + 1, n, 2).copy())


    @classmethod
    def acceptance9_snapshot(cls, index, H=60):
        """Snapshot `index` of acceptance criterion 9's random sequence
        (tests/acceptance_test.cpp:271-334: mt19937_64(4242))."""
        cap = 2 * (H + 1) * 16
        field = np.zeros(cap)
        warm = np.zeros(18)
        wl = C.c_int32()
        s = abi.pp_snapshot()
        n = cls.lib().ref_acceptance9_snapshot(index, H, C.byref(s), _ptr(field), cap,
                                               _ptr(warm), C.byref(wl))
        if n < 0:
            raise RuntimeError(cls.lib().ref_last_error().decode())
        return abi.Snapshot(ev=(s.ev_x, s.ev_y, s.ev_phi, s.ev_v),
                            actuator_delta=s.actuator_delta, prev_action=(s.prev_a0, s.prev_a1),
                            goal=(s.goal_x, s.goal_y, s.goal_phi, s.goal_v),
                            field=field[: 2 * (H + 1) * n].reshape(H + 1, n, 2).copy(),
                            warm_theta=warm.copy() if wl.value else None)


class Port(_Base):
    """The plain-C restatement (paraplan_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not PORT_SO.exists():
                raise FileNotFoundError(f"{PORT_SO} missing: run `make -C oracle`")
            L = C.CDLL(str(PORT_SO))
            L.po_param_count.argtypes = [C.POINTER(abi.pp_model)]
            L.po_validate.argtypes = [C.POINTER(abi.pp_model), C.c_char_p, C.c_int32]
            L.po_sample_candidate.argtypes = [C.POINTER(abi.pp_model), C.POINTER(C.c_double),
                                              C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
                                              C.POINTER(C.c_double)]
            L.po_rollout.argtypes = [C.POINTER(abi.pp_model), C.POINTER(abi.pp_snapshot),
                                     C.POINTER(C.c_double), C.POINTER(abi.pp_rollout_stats),
                                     C.POINTER(C.c_double), C.POINTER(C.c_int32)]
            L.po_eval_candidates.argtypes = [C.POINTER(abi.pp_model), C.POINTER(abi.pp_snapshot),
                                             C.c_uint64, C.c_int32, C.c_int32,
                                             C.POINTER(C.c_double), C.c_int64, C.c_int64,
                                             C.c_void_p]
            L.po_eval_candidates_mt.argtypes = [C.POINTER(abi.pp_model),
                                                C.POINTER(abi.pp_snapshot), C.c_uint64,
                                                C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                                C.c_int64, C.c_int64, C.c_int32, C.c_void_p]
            L.po_plan_step.argtypes = [C.POINTER(abi.pp_model), C.POINTER(abi.pp_snapshot),
                                       C.c_uint64, C.c_int32, C.POINTER(abi.pp_plan_output)]
            L.po_rng_stream.argtypes = [C.c_uint64] * 5 + [C.c_int32, C.c_int32, C.c_void_p]
            L.po_better.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_double,
                                    C.c_double]
            cls._lib = L
        return cls._lib

    def __init__(self, model: abi.Model):
        self.model = model
        self._m = model.to_c()
        msg = C.create_string_buffer(256)
        if self.lib().po_validate(C.byref(self._m), msg, 256) != 0:
            raise ValueError(msg.value.decode())
        self.n_params = self.lib().po_param_count(C.byref(self._m))

    def plan_step(self, snap, t, threads=1):
        s = snap.to_c(self.model.H)
        o, theta, traj = abi.plan_output_buffers(self.n_params, self.model.H)
        if self.lib().po_plan_step(C.byref(self._m), C.byref(s), t, threads, C.byref(o)) != 0:
            raise ValueError("warm start vector size mismatch")
        return o, theta, traj[: o.trajectory_len].copy()

    def rollout(self, snap, theta):
        s = snap.to_c(self.model.H)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        st = abi.pp_rollout_stats()
        traj = np.zeros((self.model.H + 1, 4))
        n = C.c_int32()
        self.lib().po_rollout(C.byref(self._m), C.byref(s), _ptr(th), C.byref(st), _ptr(traj),
                              C.byref(n))
        return st, traj[: n.value].copy()

    def sample_candidate(self, center, t, restart, it, cand):
        c = np.ascontiguousarray(center, dtype=np.float64)
        out = np.zeros_like(c)
        self.lib().po_sample_candidate(C.byref(self._m), _ptr(c), t, restart, it, cand, _ptr(out))
        return out

    def eval_candidates(self, snap, t, it, restart, center, c_begin, c_end, threads=None):
        """Per-candidate stats; threads=None uses every host core (the bits do
        not depend on the thread count)."""
        s = snap.to_c(self.model.H)
        c = np.ascontiguousarray(center, dtype=np.float64)
        out = self._stats_array(c_end - c_begin)
        n = (os.cpu_count() or 1) if threads is None else threads
        if c_end - c_begin < 256:
            n = 1
        self.lib().po_eval_candidates_mt(C.byref(self._m), C.byref(s), t, it, restart, _ptr(c),
                                         c_begin, c_end, n, out.ctypes.data)
        return out

    @classmethod
    def rng_stream(cls, key, kind, n):
        out = np.zeros(n, dtype=np.uint64 if kind == 0 else np.float64)
        cls.lib().po_rng_stream(*key, kind, n, out.ctypes.data)
        return out
