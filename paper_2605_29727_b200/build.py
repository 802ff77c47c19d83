"""In-tree build of libbastion.so (sm_100a) with plain nvcc.

The shared library has a C ABI only (include/bastion.h) — no torch, no
pybind — so it loads with ctypes and travels to the GPU box as a file.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# measurement builds go to their own directory / library (load with BASTION_LIB=...):
# BST_TRACE=1 -> libbastion_trace.so; BST_BUILD_TAG=x with BST_NVCC_EXTRA="-D..." -> libbastion_x.so
_TAG = "trace" if os.environ.get("BST_TRACE") == "1" else os.environ.get("BST_BUILD_TAG", "")
BUILD = PKG / (f"_build_{_TAG}" if _TAG else "_build")
LIB = PKG / (f"libbastion_{_TAG}.so" if _TAG else "libbastion.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
TRACE = ["-DBST_TRACE"] if os.environ.get("BST_TRACE") == "1" else []  # phase tracing builds
TRACE += os.environ.get("BST_NVCC_EXTRA", "").split() if os.environ.get("BST_BUILD_TAG") else []
BASE = TRACE + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}",
        "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr", "-diag-suppress", "550,177"]
# fp64 controller arithmetic must not be contracted into FMAs (bit parity with Python floats)
PER_FILE = {"expand.cu": ["-fmad=false"]}


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _deps() -> list[Path]:
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))


def _stale(obj: Path, src: Path, dep_mtime: float) -> bool:
    return not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, dep_mtime)


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    dep_mtime = max((p.stat().st_mtime for p in _deps()), default=0.0)
    srcs = _sources()
    objs = [BUILD / (s.stem + ".o") for s in srcs]

    def compile_one(pair):
        src, obj = pair
        if not _stale(obj, src, dep_mtime):
            return None
        cmd = [nvcc, *ARCH, *BASE, *PER_FILE.get(src.name, []), "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        return src.name

    with ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(compile_one, zip(srcs, objs)))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
