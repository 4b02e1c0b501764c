"""In-tree build of the CUDA library (sm_100a) -- invoked by __graft_entry__.build()."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libheddle_place.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    try:
        import nvidia.nccl
        return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    except Exception:
        return os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                            "site-packages", "nvidia", "nccl")


NCCL = _nccl_dir()
NCCL_FLAGS = ["-I", os.path.join(NCCL, "include"), "-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2",
              "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-warn-spills", "-cudart", "shared"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return (sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(glob.glob(os.path.join(CSRC, "*.h")))
            + [os.path.join(INCLUDE, "heddle_place.h"), __file__])


STAMP = LIB + ".stamp"


def digest() -> str:
    h = hashlib.sha256()
    for f in deps():
        h.update(os.path.relpath(f, ROOT).encode())
        h.update(open(f, "rb").read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def stale() -> bool:
    """Content-hash check (file mtimes change when the tree is copied to a GPU box)."""
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    return open(STAMP).read().strip() != digest()


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit (heddle_place.cu and the inst_*.cu kernel families) in
    parallel, then link the shared library."""
    if not force and not stale():
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", INCLUDE, "-I", os.path.join(NCCL, "include")]
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.splitext(os.path.basename(src))[0] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *inc, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    failed = [cmd for p, cmd in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", LIB, *objs, *NCCL_FLAGS]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    with open(STAMP, "w") as f:
        f.write(digest())
    return LIB


def build_checked(out: str) -> str:
    """Debug build with shared-memory bounds checks (-DHEDDLE_CHECK_BOUNDS), one translation unit
    (-DHEDDLE_UNITY) so that every kernel counts into the same device-side violation counter."""
    cmd = [NVCC, *ARCH, *FLAGS, "-DHEDDLE_CHECK_BOUNDS", "-DHEDDLE_UNITY", "-I", INCLUDE, "-shared", "-o", out,
           os.path.join(CSRC, "heddle_place.cu"), *NCCL_FLAGS]
    subprocess.check_call(cmd)
    return out
