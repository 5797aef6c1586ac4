"""Build libpolar.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

``python -m paper_2603_11438_b200.build`` or ``build()``; incremental (objects
under build/ are reused when newer than every source/header).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libpolar.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2,-Wall", "-I", INCLUDE, "-I", CSRC]
CU_FLAGS = ARCH + COMMON + ["-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


def _obj(src):
    return os.path.join(BUILD, os.path.basename(src) + ".o")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose):
    obj = _obj(src)
    if src.endswith(".cu"):
        cmd = [NVCC] + CU_FLAGS + ["-c", src, "-o", obj]
    else:
        cmd = [NVCC] + ARCH + COMMON + ["-x", "c++", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    log = os.path.join(BUILD, os.path.basename(src) + ".ptxas.txt")
    with open(log, "w") as f:
        f.write(r.stderr)
    if verbose:
        print(f"[build] {os.path.basename(src)}", file=sys.stderr)
    return obj


def build(verbose: bool = True, force: bool = False, defines=(), lib=None, build_dir=None) -> str:
    """defines: extra -D flags (tuning variants); lib/build_dir: alternate outputs."""
    global BUILD, LIB, CU_FLAGS, COMMON
    if defines or lib or build_dir:
        BUILD = build_dir or BUILD
        LIB = lib or LIB
        extra = [f"-D{d}" for d in defines]
        CU_FLAGS = CU_FLAGS + extra
        COMMON = COMMON + extra
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    hdrs = _headers()
    todo = [s for s in srcs if force or _stale(_obj(s), [s] + hdrs)]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
            list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [_obj(s) for s in srcs]
    if force or todo or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread",
                                                              "-Xlinker", "-soname=libpolar.so"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        if verbose:
            print(f"[build] linked {LIB}", file=sys.stderr)
    if LIB == os.path.join(PKG, "libpolar.so"):
        build_tuner(verbose, force)
    return LIB


TUNER_SRC = os.path.join(CSRC, "nccl_tuner", "tuner.cpp")
TUNER_LIB = os.path.join(PKG, "libpolar_nccl_tuner.so")


def build_tuner(verbose: bool = True, force: bool = False) -> str:
    """The NCCL tuner-plugin shim (csrc/nccl_tuner/tuner.cpp): a host-only .so
    that links libpolar.so (rpath $ORIGIN) and exports ncclTunerPlugin_v3/_v4."""
    if force or _stale(TUNER_LIB, [TUNER_SRC, LIB, os.path.join(INCLUDE, "polar.h")]):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-fvisibility=hidden", "-I", INCLUDE,
               "-I", "/usr/local/cuda/include", TUNER_SRC, "-o", TUNER_LIB, "-L", PKG, "-l:libpolar.so",
               "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"tuner build failed:\n{r.stderr}")
        if verbose:
            print(f"[build] linked {TUNER_LIB}", file=sys.stderr)
    return TUNER_LIB


if __name__ == "__main__":
    # python -m paper_2603_11438_b200.build [--force] [--variant NAME -DX=1 ...]
    argv = sys.argv[1:]
    if "--variant" in argv:
        name = argv[argv.index("--variant") + 1]
        defs = [a[2:] for a in argv if a.startswith("-D")]
        build(force=True, defines=defs, lib=os.path.join(ROOT, "build", f"variants/libpolar_{name}.so"),
              build_dir=os.path.join(ROOT, "build", f"obj_{name}"))
    else:
        build(force="--force" in argv)
