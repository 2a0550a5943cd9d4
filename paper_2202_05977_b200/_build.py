"""Build libkmd.so (the C-ABI library) in-tree with nvcc for sm_100a.

Explicit nvcc invocation (no torch JIT cache): the .so lands next to this file
so it travels to the GPU box with the repo snapshot and is the file the tests
and the bench load.  No fast-math: the kernels rely on IEEE expf / division
(DESIGN.md §5).
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libkmd.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2,-Wall",
              "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libkmd (no CPU fallback exists)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(
        os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "kmd.h")]


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


CHECKED_LIB = os.path.join(PKG, "libkmd_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Build libkmd.so, or (checked=True) libkmd_checked.so: the same sources
    with -DKMD_CHECKS (device-side bounds assertions, kmd_common.cuh)."""
    lib = CHECKED_LIB if checked else LIB
    if not (force or (is_stale() if not checked else not os.path.exists(lib) or
                      any(os.path.getmtime(p) > os.path.getmtime(lib) for p in _deps()))):
        return lib
    nvcc = nvcc_path()
    objs = []
    log_lines = []
    build_dir = os.path.join(PKG, "build_checked" if checked else "build")
    os.makedirs(build_dir, exist_ok=True)
    extra = ["-DKMD_CHECKS"] if checked else []
    def compile_one(src):
        obj = os.path.join(build_dir, os.path.basename(src)[:-3] + ".o")
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        return src, obj, cmd, subprocess.run(cmd, capture_output=True, text=True)

    # the translation units compile concurrently (one nvcc process each)
    from concurrent.futures import ThreadPoolExecutor
    srcs = sources()
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, srcs))
    for src, obj, cmd, r in results:
        log_lines.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log_lines.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link of libkmd.so failed")
    os.replace(tmp, lib)
    with open(os.path.join(build_dir, "build.log"), "w") as f:
        f.write("\n".join(log_lines))
    if verbose:
        print("\n".join(log_lines))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
