"""Build recipe for libbsp.so (sm_100a CUDA kernels + host C++ + C ABI).

Compiles every source under ``csrc/`` with nvcc (``.cu``: device code for
``-gencode arch=compute_100a,code=sm_100a``; ``.cpp``: host C++20 with
OpenMP) and links them into ``paper_2507_21253_b200/libbsp.so`` in-tree, so
the library travels to the GPU box with the repository snapshot.

Usage: ``python -m paper_2507_21253_b200.build`` (also called by
``__graft_entry__.build()``).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libbsp.so"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}", f"-I{CSRC}"]
CU_FLAGS = ARCH + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"] + COMMON
CPP_FLAGS = COMMON + ["-Xcompiler", "-fopenmp", "-Xcompiler", "-ffp-contract=off"]


def _deps_mtime() -> float:
    hdrs = list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return max((p.stat().st_mtime for p in hdrs), default=0.0)


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.name + ".o")
    dep_t = max(_deps_mtime(), src.stat().st_mtime, Path(__file__).stat().st_mtime)
    if obj.exists() and obj.stat().st_mtime >= dep_t:
        return obj
    flags = CU_FLAGS if src.suffix == ".cu" else CPP_FLAGS
    cmd = [NVCC, *flags, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":
        cmd = [NVCC, "-x", "c++", *flags, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = OBJ / (src.name + ".log")
    log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed on {src.name}")
    if verbose:
        sys.stderr.write(f"[build] {src.name}\n")
    return obj


def build(verbose: bool = True, jobs: int | None = None) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-Xcompiler", "-fopenmp",
           "-lgomp", "-cudart", "static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("link of libbsp.so failed")
    if verbose:
        sys.stderr.write(f"[build] linked {LIB}\n")
    return LIB


if __name__ == "__main__":
    build()
