"""ctypes binding of the C-ABI (include/paraplan_cuda.h) in lib/libparaplan.so.

This is the Python-side plugin surface the tests, the benchmark and the
multi-GPU shard driver use. It loads the in-tree library and fails loudly
when it is missing -- there is no CPU fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import abi

# PARAPLAN_LIB selects an alternative build (A/B experiments only)
LIB_PATH = Path(os.environ.get("PARAPLAN_LIB")
                or Path(__file__).resolve().parent / "lib" / "libparaplan.so")
_lib = None


class PlannerError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1904_06680_b200.build` "
                "(the B200 planner has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        P = C.POINTER
        L.pp_abi_version.restype = C.c_int32
        L.pp_last_error.restype = C.c_char_p
        L.pp_device_count.restype = C.c_int32
        L.pp_create.argtypes = [P(abi.pp_model), P(C.c_void_p)]
        L.pp_destroy.argtypes = [C.c_void_p]
        L.pp_param_count.argtypes = [C.c_void_p]
        L.pp_param_count.restype = C.c_int32
        L.pp_plan_step.argtypes = [C.c_void_p, P(abi.pp_snapshot), C.c_uint64, P(abi.pp_plan_output)]
        L.pp_rollout.argtypes = [C.c_void_p, P(abi.pp_snapshot), P(C.c_double), C.c_int32,
                                 P(abi.pp_rollout_stats), P(C.c_double), C.c_int32, P(C.c_int32)]
        L.pp_sample_candidate.argtypes = [C.c_void_p, P(C.c_double), C.c_int32, C.c_uint64,
                                          C.c_int32, C.c_int32, C.c_int32, P(C.c_double)]
        L.pp_perturbation_sigma.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_int32,
                                            C.c_int32]
        L.pp_perturbation_sigma.restype = C.c_double
        L.pp_upload_snapshot.argtypes = [C.c_void_p, P(abi.pp_snapshot)]
        L.pp_plan_step_points.argtypes = [C.c_void_p, P(abi.pp_snapshot_points), C.c_uint64,
                                          P(abi.pp_plan_output)]
        L.pp_upload_points.argtypes = [C.c_void_p, P(abi.pp_snapshot_points)]
        L.pp_draw_theta.argtypes = [C.c_void_p, P(C.c_double), C.c_int32, C.c_uint64, C.c_int32,
                                    C.c_int32, C.c_int64, C.c_int64, P(C.c_double)]
        L.pp_evaluate.argtypes = [C.c_void_p, P(abi.pp_snapshot), C.c_uint64, C.c_int32, C.c_int32,
                                  C.c_int32, P(C.c_double), C.c_int64, C.c_int64, C.c_void_p,
                                  C.c_void_p]
        L.pp_eval_theta.argtypes = [C.c_void_p, P(abi.pp_snapshot), P(C.c_double), C.c_int64,
                                    C.c_void_p]
        L.pp_merge_records.argtypes = [C.c_void_p, C.c_int32, P(abi.pp_record)]
        L.pp_key_better.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_double,
                                    C.c_double]
        L.pp_key_better.restype = C.c_int32
        L.pp_last_timing.argtypes = [C.c_void_p, P(abi.pp_timing)]
        L.pp_stream.argtypes = [C.c_void_p]
        L.pp_stream.restype = C.c_void_p
        L.pp_measure_fp32_peak.argtypes = [C.c_int32, P(C.c_double), P(C.c_double)]
        L.pp_comm_unique_id.argtypes = [C.c_char_p]
        L.pp_comm_init.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_int32]
        L.pp_exchange_kind.argtypes = [C.c_void_p]
        L.pp_exchange_kind.restype = C.c_char_p
        L.pp_pack_key.argtypes = [C.c_int32, C.c_int32, C.c_float, C.c_uint32]
        L.pp_pack_key.restype = C.c_uint64
        L.pp_unpack_key.argtypes = [C.c_uint64, P(C.c_int32), P(C.c_int32), P(C.c_float),
                                    P(C.c_uint32)]
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    """Every entry point include/paraplan_cuda.h declares."""
    return ["pp_create", "pp_destroy", "pp_last_error", "pp_param_count", "pp_abi_version",
            "pp_plan_step", "pp_plan_step_points", "pp_upload_points", "pp_draw_theta", "pp_rollout", "pp_sample_candidate", "pp_perturbation_sigma",
            "pp_upload_snapshot", "pp_evaluate", "pp_eval_theta", "pp_merge_records",
            "pp_key_better", "pp_last_timing", "pp_stream", "pp_device_count",
            "pp_measure_fp32_peak", "pp_comm_unique_id", "pp_comm_init", "pp_exchange_kind",
            "pp_pack_key", "pp_unpack_key"]


def _check(rc: int):
    if rc != 0:
        msg = lib().pp_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise PlannerError(msg)


def device_count() -> int:
    return lib().pp_device_count()


def merge_records(recs: np.ndarray) -> np.ndarray:
    recs = np.ascontiguousarray(recs, dtype=abi.RECORD_DTYPE)
    out = abi.pp_record()
    _check(lib().pp_merge_records(recs.ctypes.data, len(recs), C.byref(out)))
    return np.array([(out.cls, out.candidate, out.restart, out.iter, out.k1, out.k2)],
                    dtype=abi.RECORD_DTYPE)[0]


def measure_fp32_peak(device: int = 0) -> tuple[float, float]:
    tf, mhz = C.c_double(), C.c_double()
    _check(lib().pp_measure_fp32_peak(device, C.byref(tf), C.byref(mhz)))
    return tf.value, mhz.value


def comm_unique_id() -> bytes:
    """NCCL unique id for pp_comm_init (rank 0 makes it, the caller shares it)."""
    buf = C.create_string_buffer(128)
    _check(lib().pp_comm_unique_id(buf))
    return buf.raw


def pack_key(cls: int, t_goal: int, cost: float, candidate: int) -> int:
    """The packed winner key of the cross-GPU allreduce (keypack.h)."""
    return lib().pp_pack_key(cls, t_goal, cost, candidate)


def unpack_key(key: int) -> tuple[int, int, float, int]:
    c, tg, cost, idx = C.c_int32(), C.c_int32(), C.c_float(), C.c_uint32()
    lib().pp_unpack_key(key, C.byref(c), C.byref(tg), C.byref(cost), C.byref(idx))
    return c.value, tg.value, cost.value, idx.value


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class DevicePlanner:
    """One pp_handle: one GPU, one stream. Mirrors the reference Planner."""

    def __init__(self, model: abi.Model):
        self.model = model
        self._m = model.to_c()
        h = C.c_void_p()
        _check(lib().pp_create(C.byref(self._m), C.byref(h)))
        self.h = h
        self.n_params = lib().pp_param_count(self.h)

    def close(self):
        if getattr(self, "h", None):
            lib().pp_destroy(self.h)
            self.h = None

    __del__ = close

    def plan_step(self, snap: abi.Snapshot, t: int):
        s = snap.to_c(self.model.H)
        o, theta, traj = abi.plan_output_buffers(self.n_params, self.model.H)
        _check(lib().pp_plan_step(self.h, C.byref(s), t, C.byref(o)))
        return o, theta, traj[: o.trajectory_len].copy()

    def draw_theta(self, center, t: int, restart: int, iter_: int, c0: int, c1: int):
        """The device's theta draws for candidates [c0, c1) (RNG parity dump)."""
        ctr = np.ascontiguousarray(center, dtype=np.float64)
        out = np.zeros((max(c1 - c0, 0), self.n_params))
        _check(lib().pp_draw_theta(self.h, ctr.ctypes.data_as(C.POINTER(C.c_double)), len(ctr), t,
                                   restart, iter_, c0, c1,
                                   out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def plan_step_points(self, snap: abi.Snapshot, points, t: int, T_s: float = 0.1):
        """plan_step on extrapolate(points): raw anchor-frame points (N, 4)."""
        s = abi.points_snapshot(snap, points, T_s)
        o, theta, traj = abi.plan_output_buffers(self.n_params, self.model.H)
        _check(lib().pp_plan_step_points(self.h, C.byref(s), t, C.byref(o)))
        return o, theta, traj[: o.trajectory_len].copy()

    def upload(self, snap: abi.Snapshot):
        s = snap.to_c(self.model.H)
        _check(lib().pp_upload_snapshot(self.h, C.byref(s)))

    def evaluate(self, snap: abi.Snapshot | None, t: int, it: int, r0: int, rc: int, center,
                 c0: int, c1: int, per_sample: bool = False):
        s = snap.to_c(self.model.H) if snap is not None else None
        c = np.ascontiguousarray(center if center is not None else np.zeros(self.n_params),
                                 dtype=np.float64)
        recs = np.zeros(rc, dtype=abi.RECORD_DTYPE)
        ps = np.zeros(rc * max(c1 - c0, 0), dtype=abi.STATS_DTYPE) if per_sample else None
        _check(lib().pp_evaluate(self.h, C.byref(s) if s is not None else None, t, it, r0, rc,
                                 _dptr(c), c0, c1, recs.ctypes.data,
                                 ps.ctypes.data if ps is not None else None))
        return recs, ps

    def eval_theta(self, snap: abi.Snapshot, theta: np.ndarray):
        s = snap.to_c(self.model.H)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        out = np.zeros(th.shape[0], dtype=abi.STATS_DTYPE)
        _check(lib().pp_eval_theta(self.h, C.byref(s), _dptr(th), th.shape[0], out.ctypes.data))
        return out

    def rollout(self, snap: abi.Snapshot, theta):
        s = snap.to_c(self.model.H)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        st = abi.pp_rollout_stats()
        traj = np.zeros((self.model.H + 1, 4))
        n = C.c_int32()
        _check(lib().pp_rollout(self.h, C.byref(s), _dptr(th), len(th), C.byref(st), _dptr(traj),
                                self.model.H + 1, C.byref(n)))
        return st, traj[: n.value].copy()

    def perturbation_sigma(self, t, restart, it, cand) -> float:
        return lib().pp_perturbation_sigma(self.h, t, restart, it, cand)

    def sample_candidate(self, center, t, restart, it, cand):
        c = np.ascontiguousarray(center, dtype=np.float64)
        out = np.zeros_like(c)
        _check(lib().pp_sample_candidate(self.h, _dptr(c), len(c), t, restart, it, cand,
                                         _dptr(out)))
        return out

    def join_communicator(self, unique_id: bytes, world: int, rank: int):
        """This planner becomes rank `rank` of `world` (one process per GPU):
        plan_step evaluates its shard and exchanges over NCCL."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        _check(lib().pp_comm_init(self.h, unique_id, world, rank))

    def exchange(self) -> str:
        return lib().pp_exchange_kind(self.h).decode()

    def timing(self) -> abi.pp_timing:
        t = abi.pp_timing()
        _check(lib().pp_last_timing(self.h, C.byref(t)))
        return t

    def stream(self) -> int:
        return lib().pp_stream(self.h) or 0
