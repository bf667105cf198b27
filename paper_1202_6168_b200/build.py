"""Build libditer.so in-tree with nvcc for sm_100a (B200) only.

    python -m paper_1202_6168_b200.build [--force]

The library links NCCL when its header is found (multi-GPU exchange) and the
static CUDA runtime; the output lands next to this file so it travels with
the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libditer.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "diter.h"), os.path.abspath(__file__)]


def _nccl_flags():
    """NCCL for the multi-GPU exchange.  Prefer the NCCL wheel torch itself loads
    (nvidia/nccl in site-packages, with an rpath to it): both libraries then resolve
    the one libnccl.so.2 whichever is loaded first -- linking the older system copy
    let libditer pull it in before torch, whose libtorch_cuda then misses newer NCCL
    symbols.  Else the system header + library, else none."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for root in (spec.submodule_search_locations or []) if spec else []:
            inc, lib = os.path.join(root, "include"), os.path.join(root, "lib")
            if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
                return (["-DDITER_WITH_NCCL=1", "-I", inc],
                        ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib])
    except Exception:
        pass
    inc = "/usr/include/nccl.h"
    lib = "/usr/lib/x86_64-linux-gnu/libnccl.so"
    if os.path.exists(inc) and os.path.exists(lib):
        return ["-DDITER_WITH_NCCL=1"], ["-lnccl"]
    return [], []


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    cflags, lflags = _nccl_flags()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v" if verbose else "-O3",
           "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), *cflags,
           "-o", SO + ".tmp", *_sources(), *lflags]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
