"""Build the in-tree CUDA library `libsosadmm.so` for sm_100a (explicit nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsosadmm.so")
SOURCES = ["sosadmm.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for c in [os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"]:
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(HERE, "..", "include", "sosadmm.h")]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def _nccl_include() -> list:
    """nccl.h of the NCCL that torch loads (the nvidia-nccl wheel); only types are used at compile
    time, the library is resolved at run time with dlopen (csrc/sosadmm.cu)."""
    try:
        import nvidia.nccl  # noqa: F401

        d = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return ["-I", d]
    except Exception:
        pass
    return []


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    extra = os.environ.get("SOSADMM_NVCC_EXTRA", "").split()  # experiments only (e.g. -DTRD_SUSPEND_NS=...)
    cmd = [_nvcc()] + NVCC_FLAGS + extra + _nccl_include() + ["-o", LIB] + [os.path.join(CSRC, s) for s in SOURCES] + ["-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
