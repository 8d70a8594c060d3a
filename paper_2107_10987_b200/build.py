"""Build libomb200.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

-fmad=false keeps every a*b+c as two rounded operations like the reference
(FMA-free x86-64 build); explicit __fma_rn() calls are not
affected.  -lineinfo maps ncu source counters back to omb_stage.cuh.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libomb200.so")
SOURCES = ["omb_kernels.cu", "omb_fmm.cu"]
HEADERS = ["omb_math.cuh", "omb_stage.cuh", "omb_pow.cuh", "omb_pow_tables.cuh", "omb_items.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
              "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC"]


def _stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "omb200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, out=None, defines=()):
    so = out or SO
    if not force and out is None and not _stale():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-o", so] + [os.path.join(CSRC, s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libomb200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    return so


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
