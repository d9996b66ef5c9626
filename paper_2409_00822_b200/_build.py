"""Build recipe for librtk.so (sm_100a).  Used by __graft_entry__.build() and tests.

Flags: -fmad=false -ftz=false -prec-div=true and no fast-math, so every fp32
operation is one IEEE round-to-nearest op with subnormals preserved -- the
numeric contract of the reference kernels (_kernels.py:1-10)."""

from __future__ import annotations

import fcntl
import os
import shutil
import subprocess
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "librtk.so")
# one translation unit per mode so nvcc compiles the kernel instantiations in parallel
SOURCES = [os.path.join(CSRC, f) for f in ("rtk_dispatch_exact.cu", "rtk_dispatch_early.cu", "rtk_dispatch_trace.cu",
                                           "rtk_dispatch_x16.cu", "rtk_dispatch_maxk.cu", "rtk_capi.cu", "rtk_maxk.cu", "rtk_io.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("rtk_kernels.cuh", "rtk_pair.cuh", "rtk_big.cuh", "rtk_block.cuh",
                                                  "rtk_dispatch.cuh")] + [os.path.join(ROOT, "include", "rtk.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xcompiler", "-pthread",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise FileNotFoundError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra: list[str] | None = None) -> str:
    """Compile librtk.so (or a variant at `out` with extra nvcc flags, e.g.
    ["-DRTK_L2_AHEAD=4"], for tuning sweeps)."""
    target = out or SO
    if out is None and not force and not needs_build():
        return SO
    # one builder at a time (every torchrun rank calls this); the others wait
    # and then find the library current
    with open(target + ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        try:
            if out is None and not force and not needs_build():
                return SO
            return _compile(target, verbose, extra)
        finally:
            fcntl.flock(lock, fcntl.LOCK_UN)


def _compile(target: str, verbose: bool, extra: list[str] | None) -> str:
    tmp = f"{target}.tmp.{os.getpid()}"
    inc = ["-I", os.path.join(ROOT, "include")]
    with tempfile.TemporaryDirectory(prefix="rtk_build_") as objdir:
        procs, objs = [], []
        for src in SOURCES:
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            cmd = [nvcc(), *NVCC_FLAGS, *(extra or []), *inc, "-c", "-o", obj, src]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((subprocess.Popen(cmd), cmd))
            objs.append(obj)
        failed = [cmd for p, cmd in procs if p.wait() != 0]
        if failed:
            raise subprocess.CalledProcessError(1, failed[0])
        link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-pthread",
                "-o", tmp, *objs]
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.run(link, check=True)
    os.replace(tmp, target)
    return target
