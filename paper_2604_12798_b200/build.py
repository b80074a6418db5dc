"""Build libvfa_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""

from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "vfa_fwd.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("ptx.cuh", "schedule.h")] + [
    os.path.join(ROOT, "include", "vfa_b200.h")]
OUT = os.path.join(HERE, "libvfa_b200.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(s) <= t for s in DEPS)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """Build libvfa_b200.so (trace=True: libvfa_b200_trace.so with the -DVFA_TRACE debug
    timeline compiled in, for scripts/trace_timeline.py; never the product library)."""
    out = OUT.replace(".so", "_trace.so") if trace else OUT
    if not force and up_to_date(out):
        return out
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DVFA_TRACE"] if trace else []), "-o", out + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import sys
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
