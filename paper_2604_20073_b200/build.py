"""Build libsrdl.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_2604_20073_b200.build [--force]

The shared object lands next to this file so it travels with the source
tree to the GPU box; nothing is installed into site-packages.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libsrdl.so")
SOURCES = ["scan.cu", "sort.cu", "setops.cu", "hashset.cu", "wcoj.cu", "wcoj_mode0.cu", "wcoj_mode1.cu",
           "wcoj_mode2.cu", "wcoj_jit.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
LIBS = ["-ldl"]  # NVRTC is opened with dlopen (csrc/wcoj_jit.cu)
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES]
    files += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    files += [os.path.join(INCLUDE, "srdl.h")]
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    built = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= built for f in _inputs())


def _compile_and_link(out: str, defines=(), verbose=False) -> str:
    """Each source compiled on its own thread (the WCOJ instances dominate),
    then one link into `out`."""
    from concurrent.futures import ThreadPoolExecutor

    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    objdir = os.path.join(HERE, "build", os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def one(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc, *ARCH, *FLAGS, *dflags, "-I", INCLUDE, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr[-4000:]}")
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as pool:
        objs = list(pool.map(one, SOURCES))
    tmp = out + ".tmp"
    cmd = [nvcc, *ARCH, *FLAGS, "-o", tmp, *objs, *LIBS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, out)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    return _compile_and_link(LIB, verbose=verbose)


def build_variant(name: str, defines: list) -> str:
    """libsrdl_<name>.so with extra -D flags, for A/B runs selected through
    SRDL_LIBRARY (never loaded unless asked for)."""
    return _compile_and_link(os.path.join(HERE, f"libsrdl_{name}.so"), defines)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
