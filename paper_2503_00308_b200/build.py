"""Build libabsplat.so (sm_100a) in-tree with nvcc.

Each .cu in csrc/ is compiled to an object in csrc/build/ (in parallel) and linked into
paper_2503_00308_b200/libabsplat.so with the CUDA runtime linked statically, so the library
travels to the GPU box with the repository snapshot and needs no JIT cache.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(CSRC, "build")
LIB = os.path.join(HERE, "libabsplat.so")
LIB_CHECKED = os.path.join(HERE, "libabsplat_checked.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
SOURCES = ["absplat.cu", "k_setup.cu", "k_bin.cu", "k_tile.cu", "k_concrete.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE,
         "--expt-relaxed-constexpr"] + os.environ.get("ABSPLAT_NVCC_EXTRA", "").split()


def _deps_mtime() -> float:
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))]
    files.append(os.path.join(INCLUDE, "absplat.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, bdir: str = BUILD, checked: bool = False) -> str:
    obj = os.path.join(bdir, src.replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *FLAGS, *(["-DABSPLAT_CHECKS"] if checked else []), "-c",
           os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked=True: libabsplat_checked.so with the device-side bounds checks (DCHECK) on."""
    lib = LIB_CHECKED if checked else LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= _deps_mtime():
        return lib
    bdir = BUILD + ("_checked" if checked else "")
    os.makedirs(bdir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda src: _compile(src, bdir, checked), SOURCES))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv)
