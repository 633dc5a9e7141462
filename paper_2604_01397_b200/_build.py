"""Build libexactz.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libexactz.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["exactz.cu"]
HEADERS = ["kernels.cuh", "mesh.cuh", "sharded.cuh", "stencil_fast.cuh", "stencil_key.cuh", "vulnerability.cuh", "editlog.cuh"]

FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    # IEEE-exact float semantics: the path must be bit-exact with the oracle
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xcompiler", "-Wno-deprecated-declarations",
    "-shared",
]


def _git() -> str:
    try:
        return subprocess.check_output(["git", "-C", ROOT, "describe", "--always", "--dirty"],
                                       stderr=subprocess.DEVNULL, text=True).strip()
    except Exception:
        return "nogit"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "exactz.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def _nccl_link() -> list:
    """Link the NCCL that torch bundles (nvidia-nccl wheel), with an rpath to it.

    Linking the system libnccl.so.2 (an older 2.27) made whichever library
    loaded first own the soname: loading libexactz.so before `import torch`
    left libtorch_cuda.so without the 2.28 symbols it needs."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia")
        for base in (spec.submodule_search_locations or []):
            d = os.path.join(base, "nccl", "lib")
            if os.path.exists(os.path.join(d, "libnccl.so.2")):
                return ["-L", d, "-l:libnccl.so.2", "-Xlinker", f"-rpath={d}"]
    except Exception:
        pass
    return ["-lnccl"]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, f"-DEXACTZ_GIT=\"{_git()}\"", "-I", os.path.join(ROOT, "include"),
           "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES], *_nccl_link(),
           *os.environ.get("EXACTZ_NVCC_EXTRA", "").split()]  # dev knob (tuning builds)
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv))
