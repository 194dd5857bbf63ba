"""Build the in-tree sm_100a library: lib/libforestcoll.so.

    python -m paper_2402_06787_b200.build [--force]

nvcc cross-compiles for sm_100a without a GPU.  The .so links the static
CUDA runtime and resolves driver entry points at run time, so it loads on
CPU-only machines (symbol checks) and travels to the GPU box in-tree.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "lib", "libforestcoll.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-Wall", "-shared",
    "-Xptxas", "-v",
    "-diag-suppress", "550",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def inputs():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h"))) + sorted(
        glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(REPO, "include", "forestcoll.h")]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in inputs())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit in parallel (-c), then link the .so."""
    if not force and not stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(PKG, "lib", "obj")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    procs = []
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        procs.append((src, subprocess.Popen([nvcc, *compile_flags, "-c", "-o", obj, src],
                                            stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
    log = []
    failed = False
    for src, pr in procs:
        out, err = pr.communicate()
        log.append(f"== {os.path.basename(src)}\n{out}{err}")
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(out + err)
    with open(os.path.join(PKG, "lib", "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    if failed:
        raise RuntimeError("nvcc failed building libforestcoll.so")
    tmp = OUT + ".tmp"
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                        "-Xcompiler", "-fPIC", "-o", tmp, *objs], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed for libforestcoll.so")
    if verbose:
        sys.stderr.write("\n".join(log))
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
