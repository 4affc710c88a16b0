"""CPU checks of the boundary and of the benchmark inputs.

* the C-ABI library loads and exports every entry point include/paraplan_cuda.h
  declares; the ctypes PODs have the C layout (compiled probe);
* snapshots built through this repo's host API (select_goal -> sense ->
  extrapolate) are bit-identical to the reference's for every builtin
  scenario, and the C2 fixture senses exactly 20 points, 4 moving.
"""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT
from oracle.oracle import Ref
from paper_1904_06680_b200 import abi, capi, workloads

HEADER = ROOT / "include" / "paraplan_cuda.h"


def declared_symbols() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"\b(pp_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    lib = capi.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in sorted(syms):
        assert hasattr(lib, s), f"{s} declared in paraplan_cuda.h but not exported"
    assert set(capi.exported_symbols()) == syms
    assert lib.pp_abi_version() == 2


def test_struct_layout_matches_c(tmp_path: Path):
    src = tmp_path / "probe.c"
    names = ["pp_vehicle", "pp_norm", "pp_config", "pp_model", "pp_snapshot", "pp_snapshot_points",
             "pp_rollout_stats", "pp_record", "pp_plan_output", "pp_timing"]
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "paraplan_cuda.h"\n'
                   "int main(void){\n" +
                   "".join(f'printf("%zu\\n", sizeof({n}));\n' for n in names) +
                   'printf("%zu %zu %zu\\n", offsetof(pp_snapshot, field_xy), '
                   'offsetof(pp_config, master_seed), offsetof(pp_plan_output, winner));\n'
                   "return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = [int(x) for x in out[: len(names)]]
    assert sizes == [C.sizeof(getattr(abi, n)) for n in names]
    assert int(out[-3]) == abi.pp_snapshot.field_xy.offset
    assert int(out[-2]) == abi.pp_config.master_seed.offset
    assert int(out[-1]) == abi.pp_plan_output.winner.offset


def test_create_without_gpu_reports_no_device():
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    m = abi.Model().to_c()
    h = C.c_void_p()
    rc = capi.lib().pp_create(C.byref(m), C.byref(h))
    assert rc == 4 and not h.value  # PP_NO_DEVICE, no handle, no fallback
    assert b"no CPU fallback" in capi.lib().pp_last_error()


def test_invalid_model_reports_reference_message():
    m = abi.Model(n_candidates=0).to_c()
    h = C.c_void_p()
    assert capi.lib().pp_create(C.byref(m), C.byref(h)) == 1  # PP_INVALID_ARGUMENT
    assert capi.lib().pp_last_error() == b"n must be >= 1"
    m = abi.Model(layer_sizes=(4, 2, 2)).to_c()
    assert capi.lib().pp_create(C.byref(m), C.byref(h)) == 1
    assert capi.lib().pp_last_error() == b"input layer must have 5 units"


def test_merge_records_keeps_lowest_index_on_ties():
    recs = np.array([(1, 5, 0, 0, -2.0, 0.0), (-1, -1, 0, 0, 0, 0), (1, 900, 0, 0, -2.0, 0.0),
                     (1, 1000, 0, 0, -1.5, 0.0)], dtype=abi.RECORD_DTYPE)
    m = capi.merge_records(recs[:3])
    assert m["candidate"] == 5
    assert capi.merge_records(recs)["candidate"] == 1000


@pytest.mark.parametrize("name", ["exp1", "exp2", "exp3_explicit", "exp3_auxiliary", "exp4",
                                  "exp5_3wp", "exp5_2wp"])
@pytest.mark.parametrize("t", [0, 7])
def test_builtin_snapshots_match_reference(name, t):
    H = 30
    ours = workloads.builtin_snapshot(name, t, H)
    ref = Ref.builtin_snapshot(name, t, H)
    assert ours.ev == ref.ev and ours.goal == ref.goal
    assert ours.prev_action == ref.prev_action
    assert ours.field.tobytes() == ref.field.tobytes()


def test_c2_fixture_senses_twenty_points_four_moving(pp):
    m = workloads.c2_mission()
    pts = pp.sense(m, pp.VehicleState(0, 0, 0, 0), 5, 20, 0.1)
    assert len(pts) == 20 and sum(p.speed > 0 for p in pts) == 4
    w = workloads.c2()
    assert w.snapshot.field.shape == (31, 20, 2)
    assert abs(w.snapshot.goal[0] - 30.0) < 1e-12 and w.samples == 1 << 20
    # the oncoming corners close in over the horizon (moving rows differ)
    moving = np.any(w.snapshot.field[30] != w.snapshot.field[0], axis=1)
    assert moving.sum() == 4


def test_c1_and_c4_inputs():
    w = workloads.c1()
    assert w.snapshot.field.shape == (21, 18, 2) and w.samples == 4096
    lot = workloads.densified_lot(10000)
    assert lot.shape == (10000, 4) and np.all(np.abs(lot[:, 0]) <= 6.5)


def test_algorithmic_flops_formula():
    # 48 + 2*MAC per step, 19 + 6N per checked state; MAC([5,2,2]) = 14
    assert workloads.algorithmic_flops([5, 2, 2], 20, 10, 11) == 10 * 76 + 11 * 139


def test_model_devices_field():
    """pp_config.devices (C-ABI v2): the list is copied with its length; more
    than PP_MAX_DEVICES is refused before it reaches the library."""
    c = abi.Model(devices=[3, 1]).to_c().config
    assert c.n_devices == 2 and list(c.devices)[:2] == [3, 1]
    assert abi.Model().to_c().config.n_devices == 0
    with pytest.raises(ValueError):
        abi.Model(devices=list(range(9))).to_c()
