"""Build the native libraries in-tree (no JIT cache: the .so files travel to
the GPU box with the repo snapshot).

  libqvb200.so        product: sm_100a kernels + runtime + C ABI (include/qvb200.h)
  libqvb200_plan.so   test-only: the same host planner plus a plan interpreter
                      on std::complex, used by CPU tests to check the planner's
                      slot maps without a GPU.  Never loaded by the product path.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

PRODUCT = PKG / "libqvb200.so"
PLANCHECK = PKG / "libqvb200_plan.so"

PRODUCT_SOURCES = [CSRC / "qvb200.cu", CSRC / "plan.cpp"]
PRODUCT_DEPS = PRODUCT_SOURCES + [CSRC / "kernels.cuh", CSRC / "sampling.cuh", CSRC / "plan.hpp", CSRC / "tma_pass.cuh",
                                  INCLUDE / "qvb200.h"]
PLANCHECK_SOURCES = [CSRC / "plancheck.cpp", CSRC / "plan.cpp"]
PLANCHECK_DEPS = PLANCHECK_SOURCES + [CSRC / "plan.hpp"]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    print(" ".join(str(c) for c in cmd), file=sys.stderr)
    subprocess.run([str(c) for c in cmd], check=True)


def build_product(force: bool = False, verbose_ptxas: bool = False) -> Path:
    if force or _stale(PRODUCT, PRODUCT_DEPS):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
               "-cudart", "static", f"-I{INCLUDE}", f"-I{CSRC}", "-o", PRODUCT, *PRODUCT_SOURCES]
        if verbose_ptxas:
            cmd.insert(1, "-Xptxas=-v")
        _run(cmd)
    return PRODUCT


TRACE = PKG / "libqvb200_trace.so"


def build_trace(force: bool = False) -> Path:
    """Diagnostic build: tma_pass_kernel records a %clock64 timeline of its
    first items (tools/tma_trace.py); select it with QVB200_LIB=<path>."""
    return build_variant("trace", ["QV_TMA_TRACE"], force)


def build_variant(name: str, defines: list[str], force: bool = False) -> Path:
    """Experimental build with extra -D tuning macros (QV_C128_TILE_BITS, ...),
    selected at run time with QVB200_LIB=<path>.  Used by A/B measurements."""
    target = PKG / f"libqvb200_{name}.so"
    if force or _stale(target, PRODUCT_DEPS):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
              *[f"-D{d}" for d in defines], "-cudart", "static", f"-I{INCLUDE}", f"-I{CSRC}", "-o", target,
              *PRODUCT_SOURCES])
    return target


def build_plancheck(force: bool = False) -> Path:
    if force or _stale(PLANCHECK, PLANCHECK_DEPS):
        _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", f"-I{CSRC}", "-o", PLANCHECK, *PLANCHECK_SOURCES])
    return PLANCHECK


def build(force: bool = False) -> None:
    build_product(force)
    build_plancheck(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
