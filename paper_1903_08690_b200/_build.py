"""In-tree build of the native libraries.

    libhsb200.so   CUDA kernels + C ABI (include/hsb200.h), nvcc for sm_100a
    libhsbuild.so  host index-build / data-generator helpers, g++ + OpenMP

Both land next to this file so they travel with the repo snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
REPO = os.path.dirname(HERE)
OBJ = os.path.join(REPO, "build", "obj_debug" if os.environ.get("HSB200_DEBUG", "") == "1"
                   else "obj")
DEBUG = os.environ.get("HSB200_DEBUG", "") == "1"
# HSB200_LIB_TAG: dev A/B builds (libhsb200_<tag>.so, objects in build/obj_<tag>)
TAG = os.environ.get("HSB200_LIB_TAG", "")
if TAG:
    OBJ = os.path.join(REPO, "build", "obj_" + TAG)
LIB_CUDA = os.path.join(HERE, "libhsb200_debug.so" if DEBUG else
                        ("libhsb200_%s.so" % TAG if TAG else "libhsb200.so"))
LIB_HOST = os.path.join(HERE, "libhsbuild.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: the f64 score arithmetic must round exactly where the
# reference rounds (explicit fma() calls are still fused).
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-O3", "-I", os.path.join(REPO, "include")]
if DEBUG:
    NVFLAGS += ["-DHS_DEBUG"]
NVFLAGS += os.environ.get("HSB200_EXTRA_NVFLAGS", "").split()


def _sources(ext):
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(ext))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(REPO, "include", "hsb200.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def build_cuda(verbose=False, force=False):
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources(".cu")
    hdrs = _headers()
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC] + ARCH + NVFLAGS + ["-c", s, "-o", o])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for r in ex.map(_run, jobs):
                if verbose and r.stderr:
                    print(r.stderr)
    if force or jobs or _stale(LIB_CUDA, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB_CUDA] + objs + ["-lcudart"])
    return LIB_CUDA


def build_host(force=False):
    srcs = [os.path.join(CSRC, "hostbuild.cpp"), os.path.join(CSRC, "formats.cpp")]
    if force or _stale(LIB_HOST, srcs + [os.path.join(os.path.dirname(HERE), "include", "hsformats.h")]):
        _run(["g++", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c++17",
              "-o", LIB_HOST] + srcs)
    return LIB_HOST


def build_all(verbose=False, force=False):
    build_host(force=force)
    build_cuda(verbose=verbose, force=force)


if __name__ == "__main__":
    import sys

    build_all(verbose=True, force="--force" in sys.argv)
    print("built", LIB_CUDA, LIB_HOST)
