"""Build libomnitrack.so in-tree with nvcc for sm_100a.

    python -m paper_1910_06017_b200.build [--force]

-fmad=false keeps every kernel's floating-point operation order identical to
the numpy reference (no contraction into FMA), which is what makes the
device results bit-exact.  -lineinfo maps ncu source pages to the .cu files.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libomnitrack.so")
ROOT = os.path.dirname(HERE)

SOURCES = ["ft_api.cu", "k_imaging.cu", "k_flow.cu", "k_track.cu", "k_klt.cu"]
HEADERS = ["ft_internal.cuh", "ft_tracker.cuh", "ft_klt.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "shared",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "omnitrack.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Build LIB (or, for A/B experiments, `out` with extra -D `defines`;
    load it with FT_LIB=<path>)."""
    if out is None and not force and not _stale():
        return LIB
    target = out or LIB
    tmp = target + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-o", tmp, *[os.path.join(CSRC, f) for f in SOURCES]]
    if verbose:
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-8000:]}")
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=True, out=outs[0] if outs else None,
                defines=defs))
