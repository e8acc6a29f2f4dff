"""Build the in-tree shared libraries for sm_100a.

    libnacc.so          the product: csrc/*.cu behind include/nacc.h
    libnacc_harness.so  bench/test harness (synthetic field), include/nacc_harness.h

Compiled with explicit nvcc command lines (-gencode arch=compute_100a,
code=sm_100a, -lineinfo) so the .so files travel with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
INCLUDE = os.path.join(ROOT, "include")
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libnacc.so")
DEBUG_LIB = os.path.join(PKG, "libnacc_debug.so")  # -DNACC_DEBUG=1: device preconditions checked (csrc/debug.cu)
HARNESS_LIB = os.path.join(PKG, "libnacc_harness.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
              "-Xptxas", "-O3"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _compile(src: str, extra: list[str]) -> str:
    os.makedirs(BUILD, exist_ok=True)
    tag = ("_" + hashlib.sha1(" ".join(extra).encode()).hexdigest()[:8]) if extra else ""
    obj = os.path.join(BUILD, os.path.relpath(src, CSRC).replace(os.sep, "_") + tag + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, "-c", src, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj


def _link(objs: list[str], out: str) -> None:
    # relink when any object is newer or the object set changed (other build flags)
    stamp = out + ".objs"
    listing = "\n".join(objs)
    same = os.path.exists(stamp) and open(stamp).read() == listing
    if same and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(o) for o in objs):
        return
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed for {out}:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    with open(stamp, "w") as f:
        f.write(listing)


def build(verbose: bool = False, extra: list[str] | None = None, debug: bool = True) -> tuple[str, str]:
    """libnacc.so + libnacc_harness.so (+ libnacc_debug.so, the NACC_DEBUG precondition build)."""
    extra = list(extra or [])
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hsrcs = sorted(glob.glob(os.path.join(CSRC, "harness", "*.cu")))
    dbg = extra + ["-DNACC_DEBUG=1"]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra), srcs))
        hobjs = list(ex.map(lambda s: _compile(s, extra), hsrcs))
        dobjs = list(ex.map(lambda s: _compile(s, dbg), srcs)) if debug else None
    _link(objs, LIB)
    _link(hobjs, HARNESS_LIB)
    if debug:
        _link(dobjs, DEBUG_LIB)
    if verbose:
        print(f"built {LIB} and {HARNESS_LIB}")
    return LIB, HARNESS_LIB


if __name__ == "__main__":
    build(verbose=True, extra=sys.argv[1:])
