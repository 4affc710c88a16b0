"""B200-native per-control-step sampler of arXiv 1904.06680.

The hot path (Planner::plan_step of the reference `paraplan`) runs as one
fused sm_100a kernel per sampling round behind the C-ABI in
include/paraplan_cuda.h. Entry points:

  paper_1904_06680_b200.import_paraplan()  the drop-in `paraplan` module
                                           (pybind11, reference API)
  paper_1904_06680_b200.capi               ctypes view of the C-ABI
  paper_1904_06680_b200.distributed        one-process-per-GPU sharding
  paper_1904_06680_b200.build              in-tree nvcc/g++ build
"""
from . import abi  # noqa: F401
from .python_path import import_paraplan  # noqa: F401

__all__ = ["abi", "import_paraplan"]
