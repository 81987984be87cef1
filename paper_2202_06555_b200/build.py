"""Builds the native library in-tree with nvcc (sm_100a only).

Output: paper_2202_06555_b200/libddsg_b200.so (git-ignored, travels to the
GPU box with the gpurun snapshot).  Objects go to build/ and are rebuilt only
when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# Experiment builds (A/B measurements of compile-time variants): DDSG_BUILD_TAG=t
# with DDSG_BUILD_DEFS="-DDDSG_SLOT_COLS=16 ..." compiles libddsg_b200_t.so,
# loaded with DDSG_B200_LIB=libddsg_b200_t.so (see _native.py).
BUILD_TAG = os.environ.get("DDSG_BUILD_TAG", "")
BUILD_DEFS = os.environ.get("DDSG_BUILD_DEFS", "").split()
_SUFFIX = f"_{BUILD_TAG}" if BUILD_TAG else ""
BUILD = ROOT / "build" / f"ddsg_b200{_SUFFIX}"
LIB = PKG / f"libddsg_b200{_SUFFIX}.so"
WL_SRC = PKG / "csrc_workloads" / "workloads.c"
WL_LIB = PKG / "libddsg_workloads.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "--fmad=false",  # every FP expression rounds like the reference; FMA only via __fma_rn
    "-Xcompiler",
    "-fPIC,-ffp-contract=off",
    "-Xptxas",
    "-v",
    f"-I{ROOT / 'include'}",
] + BUILD_DEFS


def _sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers() -> list[Path]:
    return sorted(list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h")))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, hdr: list[Path], verbose: bool) -> Path:
    obj = BUILD / (src.name + ".o")
    if not _stale(obj, [src, *hdr, Path(__file__)]):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":
        cmd = [NVCC, *COMMON, "-x", "c++", "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = BUILD / (src.name + ".log")
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed on {src.name}")
    if verbose:
        sys.stderr.write(f"[build] {src.name}\n")
    return obj


def build_library(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    hdr = _headers()
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), srcs))
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc link failed")
    # C++ drop-in test driver (tests/cpp): include/ddsg_b200.hpp over the C-ABI
    drv_src = ROOT / "tests" / "cpp" / "test_dropin.cpp"
    drv = ROOT / "build" / "test_dropin"
    if not BUILD_TAG and drv_src.exists() and _stale(drv, [drv_src, LIB, ROOT / "include" / "ddsg_b200.hpp"]):
        cmd = ["g++", "-std=c++20", "-O2", "-Wall", f"-I{ROOT / 'include'}", str(drv_src), f"-L{PKG}", "-lddsg_b200",
               "-Wl,-rpath,$ORIGIN/../paper_2202_06555_b200", "-o", str(drv)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("drop-in test driver build failed")
    if _stale(WL_LIB, [WL_SRC, Path(__file__)]):
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", str(WL_LIB), str(WL_SRC), "-lm"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("workloads build failed")
    return LIB


if __name__ == "__main__":
    print(build_library(verbose=True))
