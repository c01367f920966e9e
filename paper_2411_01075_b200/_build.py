"""In-tree build of the native libraries.

* ``libhet_planner.so`` — host-only C++ (g++): the planner DP core.
* ``libhetstep.so``     — sm_100a CUDA kernels + the C-ABI of
  ``include/hetstep.h`` (nvcc ``-gencode arch=compute_100a,code=sm_100a``),
  linked against the NCCL that ships with torch (nvidia-nccl wheel).

Both land in ``paper_2411_01075_b200/_lib/`` (git-ignored, travels to the GPU
box with the gpurun snapshot). Rebuilds only when a source is newer than the
library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
INCLUDE = ROOT / "include"

PLANNER_LIB = LIBDIR / "libhet_planner.so"
STEP_LIB = LIBDIR / "libhetstep.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_root() -> Path:
    import nvidia.nccl  # torch's NCCL wheel
    return Path(list(nvidia.nccl.__path__)[0])


def _stale(lib: Path, sources: list[Path]) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")


def build_planner(force: bool = False) -> Path:
    src = [CSRC / "dp_planner.cpp"]
    if force or _stale(PLANNER_LIB, src):
        LIBDIR.mkdir(exist_ok=True)
        tmp = PLANNER_LIB.with_suffix(f".tmp{os.getpid()}.so")
        _run(["g++", "-O3", "-march=x86-64-v2", "-std=c++17", "-fPIC", "-shared", "-pthread",
              *map(str, src), "-o", str(tmp)])
        os.replace(tmp, PLANNER_LIB)
    return PLANNER_LIB


def step_sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _cublas_root() -> Path:
    import nvidia.cublas  # torch's cuBLAS wheel (cuBLASLt for the epilogue GEMMs)
    return Path(list(nvidia.cublas.__path__)[0])


def build_step(force: bool = False, verbose: bool = False) -> Path:
    srcs = step_sources()
    if not (force or _stale(STEP_LIB, srcs)):
        return STEP_LIB
    LIBDIR.mkdir(exist_ok=True)
    nccl = _nccl_root()
    tmp = STEP_LIB.with_suffix(f".tmp{os.getpid()}.so")
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3",
           f"-I{INCLUDE}", f"-I{nccl / 'include'}",
           *[str(s) for s in srcs if s.suffix == ".cu"],
           f"-L{nccl / 'lib'}", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={nccl / 'lib'}",
           "-o", str(tmp)]
    _run(cmd)
    os.replace(tmp, STEP_LIB)
    return STEP_LIB


def build_all(force: bool = False) -> None:
    build_planner(force)
    build_step(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print(PLANNER_LIB, STEP_LIB)
