"""Build libvfa_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

Each translation unit (the C ABI, and one per attention variant, which instantiates that
variant's kernels) is compiled to an object in parallel, then linked into one shared
library with the CUDA runtime linked statically.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
DEPS = SOURCES + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + [
    os.path.join(ROOT, "include", "vfa_b200.h")]
OUT = os.path.join(HERE, "libvfa_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "--expt-relaxed-constexpr",
              "-diag-suppress", "177"]


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


def build(force: bool = False, verbose: bool = False, trace: bool = False, defines=()) -> str:
    """Build libvfa_b200.so (trace=True: libvfa_b200_trace.so with the -DVFA_TRACE debug
    timeline compiled in, for scripts/trace_timeline.py; never the product library).
    defines: extra -D tuning knobs for experiment builds (scripts/ab.py), which are written
    to libvfa_b200_<name>.so when `defines` is given as (name, [flags])."""
    out = OUT.replace(".so", "_trace.so") if trace else OUT
    extra = ["-DVFA_TRACE"] if trace else []
    if defines:
        name, flags = defines
        out = OUT.replace(".so", f"_{name}.so")
        extra += list(flags)
    if not force and up_to_date(out):
        return out
    objdir = os.path.join(HERE, "build", os.path.basename(out)[:-3])
    os.makedirs(objdir, exist_ok=True)
    cc = nvcc()

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [cc, *NVCC_FLAGS, *extra, *(["-Xptxas=-v"] if verbose else []), "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose:
            print(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    link = [cc, *ARCH, "-shared", "-cudart", "static", "-o", out + ".tmp", *objs]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import sys
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
