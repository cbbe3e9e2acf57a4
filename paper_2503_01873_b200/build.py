"""Build libpasa_b200.so in-tree (nvcc, sm_100a).

    python -m paper_2503_01873_b200.build        # or __graft_entry__.build()

The library is plain CUDA C++ with a C ABI (include/pasa_b200.h); the CUDA
runtime is linked statically so the .so only needs the driver at run time.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_build")
SO = os.path.join(OUT, "libpasa_b200.so")
SOURCES = ["capi.cu", "pasa_kprep.cu", "pasa_fwd.cu", "pasa_fwd_packed.cu", "pasa_gen.cu"]
HEADERS = ["sm100.cuh", "pasa_kernels.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}"]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "pasa_b200.h")]
    return any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps)


def build(verbose: bool = False, force: bool = False, trace: bool = False) -> str:
    """Build libpasa_b200.so (or, with trace=True, the clock64-timeline profiling
    variant libpasa_b200_trace.so used by tools/trace_fwd.py)."""
    out_dir = os.path.join(OUT, "trace") if trace else OUT
    so = os.path.join(OUT, "libpasa_b200_trace.so") if trace else SO
    extra = ["-DPASA_TRACE"] if trace else []
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(out_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, s):
            cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError(f"nvcc failed on {src}")
    if force or not os.path.exists(so) or any(os.path.getmtime(o) > os.path.getmtime(so) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", so, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return so


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, trace="--trace" in sys.argv))
