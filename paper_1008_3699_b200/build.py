"""Build the sm_100a shared library (C ABI of include/sweep.h) in-tree."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsweep.so")
# race-exposure variant (-DSW_JITTER, csrc/common.cuh): randomised sleeps after every barrier;
# loaded only by tests/test_gpu_jitter.py through SW_LIBRARY
LIB_JITTER = os.path.join(HERE, "libsweep_jitter.so")
SRC = os.path.join(HERE, "csrc", "sweep.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in os.listdir(d)] + [os.path.join(ROOT, "include", "sweep.h")]


def _compile(out: str, defines, verbose: bool, log: str):
    cmd = [NVCC, *FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-o", out, SRC, "-lcuda", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    with open(os.path.join(HERE, log), "w") as f:
        f.write(res.stderr)


def build(force: bool = False, verbose: bool = False, jitter: bool = True) -> str:
    """Build libsweep.so (and the race-exposure variant libsweep_jitter.so) if a source is newer."""
    newest = max(os.path.getmtime(p) for p in sources())
    extra = ["-DSW_TRACE"] if os.environ.get("SW_TRACE") == "1" else []
    extra += [f"-D{d}" for d in os.environ.get("SW_DEFINES", "").split()]
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        _compile(LIB, extra, verbose, "ptxas.log")
    if jitter and (force or not os.path.exists(LIB_JITTER) or os.path.getmtime(LIB_JITTER) < newest):
        _compile(LIB_JITTER, ["-DSW_JITTER"], False, "ptxas_jitter.log")
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
