"""In-tree build of the B200 planner (no JIT cache, no pip install).

Outputs (git-ignored, shipped to the GPU box with the snapshot):
  paper_1904_06680_b200/lib/libparaplan.so
      sm_100a kernels (nvcc -gencode arch=compute_100a,code=sm_100a) + the C-ABI
      of include/paraplan_cuda.h + the C++ API of include/paraplan/*.hpp.
      CUDA runtime linked statically.
  paper_1904_06680_b200/python/paraplan/_core<EXT_SUFFIX>
      pybind11 module, the drop-in for the reference's `paraplan._core`.

Host sources are compiled like the reference (-ffp-contract=off
-fno-math-errno) so the FP64 epilogue is bit-identical to it. The FP64
device instantiation is compiled with --fmad=false for the same reason.

Usage: python -m paper_1904_06680_b200.build [--force] [-v]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INC = ROOT / "include"
BUILD = Path(os.environ.get("PARAPLAN_BUILD_DIR", PKG / "_build"))
LIB = Path(os.environ.get("PARAPLAN_BUILD_LIB", PKG / "lib" / "libparaplan.so"))
PYPKG = PKG / "python" / "paraplan"
CORE = PYPKG / ("_core" + sysconfig.get_config_var("EXT_SUFFIX"))

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
JSON_DIRS = [
    Path(sys.prefix) / "lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann",
    Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"),
]

HOST_FLAGS = ["-std=c++20", "-O3", "-fPIC", "-fno-math-errno", "-ffp-contract=off", "-pthread",
              "-Wall", "-Wno-unused-parameter"]
# compile-time switches (PARAPLAN_NVCC_DEFS="-D..."): the -D ones reach the host
# objects too, for constants both sides share (device_api.h)
HOST_FLAGS += [d for d in os.environ.get("PARAPLAN_NVCC_DEFS", "").split() if d.startswith("-D")]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC",
              "--expt-relaxed-constexpr"] + ARCH + os.environ.get("PARAPLAN_NVCC_DEFS", "").split()


def _json_dir() -> Path:
    for d in JSON_DIRS:
        if (d / "json.hpp").exists():
            return d
    raise FileNotFoundError("nlohmann/json.hpp not found (needed by scenario.cpp)")


def _headers() -> list[Path]:
    return (sorted(INC.rglob("*.h*")) + sorted(CSRC.rglob("*.h")) + sorted(CSRC.rglob("*.hpp"))
            + sorted(CSRC.rglob("*.cuh")))


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> str:
    if verbose:
        print(" ".join(cmd), flush=True)
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"build failed:\n{' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return p.stdout + p.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    PYPKG.mkdir(parents=True, exist_ok=True)
    hdrs = _headers()
    jd = _json_dir()
    inc = [f"-I{INC}", f"-I{CSRC}", f"-I{jd}"]

    jobs = []
    objs = []
    for cu in sorted((CSRC / "cuda").glob("*.cu")):
        obj = BUILD / (cu.stem + ".o")
        objs.append(obj)
        extra = ["--fmad=false"] if cu.stem.endswith("_f64") else []
        if force or _stale(obj, [cu] + hdrs):
            jobs.append([NVCC, *NVCC_FLAGS, *extra, *inc, "-c", str(cu), "-o", str(obj)])
    for cpp in sorted((CSRC / "host").glob("*.cpp")) + sorted((CSRC / "capi").glob("*.cpp")):
        obj = BUILD / (cpp.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [cpp] + hdrs):
            jobs.append(["g++", *HOST_FLAGS, *inc, f"-I{CUDA_HOME / 'include'}", "-c", str(cpp),
                         "-o", str(obj)])
    logs = []
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for out in ex.map(lambda c: _run(c, verbose), jobs):
            logs.append(out)
    if jobs:  # keep the last compile log when nothing was stale
        (BUILD / "ptxas.log").write_text("\n".join(logs))

    if force or _stale(LIB, objs):
        _run(["g++", "-shared", "-o", str(LIB), *map(str, objs),
              f"-L{CUDA_HOME / 'lib64'}", "-lcudart_static", "-ldl", "-lrt", "-lpthread",
              "-Wl,--no-undefined"], verbose)

    if "PARAPLAN_BUILD_LIB" in os.environ:  # variant library only (A/B experiments)
        return LIB
    import pybind11
    bind = CSRC / "python" / "bindings.cpp"
    if force or _stale(CORE, [bind, LIB] + hdrs):
        py_inc = sysconfig.get_paths()["include"]
        _run(["g++", *HOST_FLAGS, "-shared", *inc, f"-I{pybind11.get_include()}", f"-I{py_inc}",
              str(bind), "-o", str(CORE), f"-L{LIB.parent}", "-lparaplan",
              "-Wl,-rpath,$ORIGIN/../../lib"], verbose)
    init = PYPKG / "__init__.py"
    init.write_text(
        '"""Online sampling in controller parameter space for vehicle motion planning\n'
        '(B200 device planner; drop-in for the reference `paraplan` package)."""\n\n'
        "from paraplan._core import *  # noqa: F401,F403\n"
        "from paraplan._core import __doc__  # noqa: F401\n\n"
        '__version__ = "0.1.0"\n')
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))


if __name__ == "__main__":
    main()
