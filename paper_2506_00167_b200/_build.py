"""Build the in-tree C-ABI library ``libcyrus_b200.so`` for sm_100a.

    python -m paper_2506_00167_b200._build [--force] [--verbose]

nvcc cross-compiles without a GPU; the .so is git-ignored but travels to the
GPU box with the repo snapshot.  No torch types cross the ABI, so the
library links only the CUDA runtime (static).
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "cyrus_b200")
LIB = os.path.join(PKG, "libcyrus_b200.so")
SOURCES = ("abi.cu", "actor.cu", "actor_gemm.cu", "actor_tc.cu", "codebook.cu", "tree.cu",
           "scheduler.cu", "ldpc.cu", "pack.cu")
HEADERS = ("cyrus_internal.cuh", "projection.cuh", "projection_lane.cuh", "actor_common.cuh")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    headers = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "cyrus_b200.h")]
    objs, jobs = [], []
    # CYR_NVCC_EXTRA: extra nvcc flags for A/B builds (e.g. -DNAME=VALUE); a
    # change of flags since the last build rebuilds every object
    extra = os.environ.get("CYR_NVCC_EXTRA", "").split()
    stamp = os.path.join(BUILD, "flags.txt")
    flags_now = " ".join(extra)
    if not os.path.exists(stamp) or open(stamp).read() != flags_now:
        force = True
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc, *ARCH, *FLAGS, *extra, "-c", s, "-o", o])

    def run(cmd):
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
        return res

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as pool:
        list(pool.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        run([nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"])
    with open(stamp, "w") as fh:
        fh.write(flags_now)
    build_fastpath(force=force, verbose=verbose)
    return LIB


FASTPATH_SRC = os.path.join(CSRC, "fastpath.c")
FASTPATH = os.path.join(PKG, "_fastpath" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def build_fastpath(force: bool = False, verbose: bool = False) -> str:
    """CPython module for the single-slot drop-in call: links the C-ABI
    library and numpy's libnpyrandom.a (bit-identical branch-noise draws)."""
    import numpy
    npyrandom = os.path.join(os.path.dirname(numpy.__file__), "random", "lib", "libnpyrandom.a")
    deps = [FASTPATH_SRC, LIB, os.path.join(INCLUDE, "cyrus_b200.h")]
    if not force and not _stale(FASTPATH, deps):
        return FASTPATH
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-std=c11", f"-I{sysconfig.get_paths()['include']}",
           f"-I{INCLUDE}", FASTPATH_SRC, f"-L{PKG}", "-lcyrus_b200", "-Wl,-rpath,$ORIGIN",
           npyrandom, "-lm", "-o", FASTPATH]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"fastpath build failed: {' '.join(cmd)}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    return FASTPATH


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
