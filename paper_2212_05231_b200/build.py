"""Build libns2b.so (sm_100a) in-tree with nvcc.

    python -m paper_2212_05231_b200.build [--force]

Each .cu compiles to an object with -gencode arch=compute_100a,code=sm_100a
-lineinfo -O3; march.cu and composite.cu additionally get -fmad=false so their
fp64 arithmetic is op-for-op with the reference's numpy (no FMA contraction).
No --use_fast_math anywhere.
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
BUILD = PKG / "_build"
LIB = PKG / "libns2b.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
NO_FMA = {"march.cu", "composite.cu", "rays.cu"}


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps_mtime():
    files = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "ns2b.h", Path(__file__)]
    return max(f.stat().st_mtime for f in files)


def _compile(src: Path, force: bool) -> Path:
    obj = BUILD / (src.stem + ".o")
    if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _deps_mtime()):
        return obj
    flags = list(COMMON) + os.environ.get("NS2B_NVCC_EXTRA", "").split()
    if src.name in NO_FMA:
        flags.append("-fmad=false")
    cmd = [NVCC, *ARCH, *flags, "-Xptxas", "-v" if os.environ.get("NS2B_PTXAS_V") else "-O3",
           "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if os.environ.get("NS2B_PTXAS_V"):
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(f".{os.getpid()}.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(tmp), *map(str, objs),
               "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
