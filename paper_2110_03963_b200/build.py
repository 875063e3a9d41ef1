"""Build libqva.so in-tree: every CUDA source compiled for sm_100a only.

    python -m paper_2110_03963_b200.build [--verbose]

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo (no fast-math: the fp64 sincos
and the FFT twiddles must keep full accuracy), linked against NCCL.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libqva.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    """Use the NCCL that torch bundles (nvidia-nccl wheel) so one libnccl.so.2 serves both
    torch.distributed and this library in the same process; fall back to the system one."""
    try:
        import nvidia.nccl as _n
        d = list(_n.__path__)[0]
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    except Exception:
        pass
    return None


NCCL_DIR = _nccl_dir()
NCCL_INC = ["-I" + os.path.join(NCCL_DIR, "include")] if NCCL_DIR else []
NCCL_LINK = (["-L" + os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2", "-Xlinker",
              "-rpath=" + os.path.join(NCCL_DIR, "lib")]
             if NCCL_DIR else ["-lnccl"])
CFLAGS = NCCL_INC + ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                 "-I" + os.path.join(os.path.dirname(HERE), "include"), "--expt-relaxed-constexpr"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(os.path.dirname(HERE), "include", "qva.h")]
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC] + CFLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            jobs.append(cmd)
    # the translation units compile independently: run them side by side
    procs = [subprocess.Popen(cmd) for cmd in jobs]
    failed = [cmd for cmd, pr in zip(jobs, procs) if pr.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    if force or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + NCCL_LINK
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    print(LIB)
