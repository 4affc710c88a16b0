"""Locate the in-tree drop-in module `paraplan` (python/paraplan/_core*.so)."""
from __future__ import annotations

import importlib
import sys
from pathlib import Path

PYDIR = Path(__file__).resolve().parent / "python"


def import_paraplan():
    if str(PYDIR) not in sys.path:
        sys.path.insert(0, str(PYDIR))
    mod = importlib.import_module("paraplan")
    if not str(Path(mod.__file__).resolve()).startswith(str(PYDIR)):
        raise ImportError(f"`paraplan` resolved to {mod.__file__}, not the in-tree B200 build")
    return mod
