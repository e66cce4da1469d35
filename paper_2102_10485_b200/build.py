"""In-tree build of the native library (sm_100a CUDA kernels + C++ host + C-ABI).

Produces paper_2102_10485_b200/_lib/libpartgan_b200.so.  Objects are rebuilt
only when a source or header is newer than the object.  cudart is linked
statically so the library does not depend on which CUDA runtime another
library in the process (e.g. torch) brought along.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
# PG_VARIANT=name PG_NVCC_DEFS="-DX=1 ..." builds a tuning variant into _lib/<name>/ (load it with PG_LIB)
VARIANT = os.environ.get("PG_VARIANT", "")
OBJ = PKG / "_lib" / (f"{VARIANT}/obj" if VARIANT else "obj")
LIB = PKG / "_lib" / (f"{VARIANT}/libpartgan_b200.so" if VARIANT else "libpartgan_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("PG_CXX", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CCBIN = ["-ccbin", CXX]
NVFLAGS = ARCH + CCBIN + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                  "-Xptxas", "-O3", f"-I{INCLUDE}"] + os.environ.get("PG_NVCC_DEFS", "").split()
# host code is compiled without FP contraction so host-side arithmetic (dataset
# generation, init) is bit-identical to the CPU oracle's
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-pthread", "-Wall", "-Wno-unused-parameter",
            "-I/usr/local/cuda/include", f"-I{INCLUDE}"]


def _headers() -> list[Path]:
    return sorted(list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h")))


def _stale(src: Path, obj: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path) -> Path:
    obj = OBJ / (src.name + ".o")
    if src.suffix == ".cu":
        cmd = [NVCC, *NVFLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = [CXX, *CXXFLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))
    deps = _headers()
    todo = [s for s in srcs if _stale(s, OBJ / (s.name + ".o"), deps)]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            for obj in ex.map(_compile, todo):
                if verbose:
                    print("built", obj.name)
    objs = [OBJ / (s.name + ".o") for s in srcs]
    if not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, *CCBIN, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs), "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
    sys.exit(0)
