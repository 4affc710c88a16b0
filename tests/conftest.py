"""Shared fixtures. `-m gpu` tests need a B200; everything else runs on CPU.

Tests compare the device planner (through the C-ABI / the drop-in module)
with the CPU checkers under oracle/ (test infrastructure only).
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1904_06680_b200 import abi  # noqa: E402

GOLDEN = ROOT / "tests" / "golden" / "reference_vectors.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100) device")


def has_gpu() -> bool:
    return os.path.exists("/dev/nvidiactl") or os.path.exists("/dev/nvidia0")


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _checkers_built():
    """Build the CPU checkers when the reference sources are present (dev
    container); on the GPU box they arrive prebuilt."""
    from oracle import oracle as orc
    if orc.REF_SRC.exists():
        orc.build()
    yield


@pytest.fixture(scope="session")
def gold():
    return json.loads(GOLDEN.read_text())


def unhex(v):
    if isinstance(v, list):
        return np.array([float.fromhex(x) for x in v], dtype=np.float64)
    return float.fromhex(v)


def golden_snapshot(gold, key) -> tuple[abi.Snapshot, int]:
    g = gold["snapshots"][key]
    shape = tuple(g["field_shape"])
    fld = unhex(g["field"]).reshape(shape) if g["field"] else np.zeros(shape)
    warm = unhex(g["warm_theta"]) if g["warm_theta"] else None
    ev = unhex(g["ev"])
    return abi.Snapshot(ev=tuple(ev), actuator_delta=unhex(g["actuator_delta"]),
                        prev_action=tuple(unhex(g["prev_action"])), goal=tuple(unhex(g["goal"])),
                        field=fld, warm_theta=warm), g["H"]


def golden_stats(rows) -> np.ndarray:
    out = np.zeros(len(rows), dtype=abi.STATS_DTYPE)
    for i, r in enumerate(rows):
        for k in abi.STATS_DTYPE.names:
            out[i][k] = r[k] if isinstance(r[k], int) else float.fromhex(r[k])
    return out


@pytest.fixture(scope="session")
def pp():
    from paper_1904_06680_b200 import import_paraplan
    return import_paraplan()
