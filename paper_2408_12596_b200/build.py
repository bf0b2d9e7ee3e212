"""In-tree build of libzp.so: sm_100a CUDA kernels + C++ host library + C ABI.

Explicit nvcc/g++ invocations (no torch JIT cache): the built .so lives in
paper_2408_12596_b200/lib/ so it travels to the GPU box with the repo snapshot.
Incremental: an object is rebuilt only when its source or any header is newer.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(PKG, "build")
LIB = os.path.join(LIBDIR, "libzp.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_HOME = os.path.dirname(os.path.dirname(NVCC))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# Host arithmetic of the planner must be bit-identical to the reference build
# (g++ -O2, no FMA contraction, no fast-math).
HOST_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
              "-Wno-unused-parameter"]
NVCC_FLAGS = ARCH + os.environ.get("ZP_EXTRA_NVCC", "").split() + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
                     "-Xptxas", "-v"] if os.environ.get("ZP_PTXAS_V") else \
    ARCH + os.environ.get("ZP_EXTRA_NVCC", "").split() + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
            "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr"]
INCLUDES = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(CSRC, "host")]


def _nccl_libdir():
    """Directory of the libnccl.so.2 that torch loads (the pip nvidia-nccl wheel): libzp links
    against the same library so torch and the runtime never load two NCCL versions."""
    try:
        import nvidia.nccl
        d = os.path.join(list(nvidia.nccl.__path__)[0], "lib")
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return d
    except Exception:
        pass
    return None


def _headers():
    hs = glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs += glob.glob(os.path.join(ROOT, "include", "*.h"))
    return hs


def _stale(obj, src, newest_header):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return os.path.getmtime(src) > t or newest_header > t


def _compile(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("compile failed: " + cmd[-1])
    return r.stdout + r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    newest = max((os.path.getmtime(h) for h in _headers()), default=0.0)
    jobs, objs = [], []
    for src in sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp"))):
        obj = os.path.join(OBJDIR, "host_" + os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(obj, src, newest):
            jobs.append(["g++"] + HOST_FLAGS + INCLUDES + ["-I", os.path.join(CUDA_HOME, "include"),
                                                          "-c", "-o", obj, src])
    for src in sorted(glob.glob(os.path.join(CSRC, "cuda", "*.cu"))):
        obj = os.path.join(OBJDIR, "cuda_" + os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(obj, src, newest):
            jobs.append([NVCC] + NVCC_FLAGS + INCLUDES + ["-c", "-o", obj, src])
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        outs = list(ex.map(_compile, jobs))
    if verbose:
        for o in outs:
            if o.strip():
                print(o)
    emap = os.path.join(CSRC, "exports.map")
    if jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs + [emap]):
        nccl = _nccl_libdir()
        nccl_flags = ["-L", nccl, "-l:libnccl.so.2", "-Xlinker", "-rpath," + nccl] if nccl else ["-lnccl"]
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + nccl_flags + [
            "-L", os.path.join(CUDA_HOME, "lib64"), "-lcudart",
            "-Xlinker", "-rpath," + os.path.join(CUDA_HOME, "lib64"), "-Xlinker", "-Bsymbolic",
            "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map")]
        _compile(cmd)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
