"""Build the in-tree native libraries with nvcc for sm_100a (no JIT cache; the .so files travel with
the repo snapshot to the GPU box).

  paper_2512_07884_b200/lib/libgspn.so   the C ABI of include/gspn.h (all CUDA kernels)
  synth/libsynth.so                      the device twin of the seeded input generator
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIBGSPN = os.path.join(LIBDIR, "libgspn.so")
SYNTH_SRC = os.path.join(ROOT, "synth", "csrc", "synth.cu")
LIBSYNTH = os.path.join(ROOT, "synth", "libsynth.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _nvcc(sources: list[str], out: str, extra: list[str] | None = None, verbose: bool = False) -> None:
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *COMMON, *(extra or []), "-o", tmp, *sources]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, out)


def build_gspn(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(glob.glob(os.path.join(CSRC, "*.h"))) + \
        [os.path.join(ROOT, "include", "gspn.h")]
    if force or _stale(LIBGSPN, deps):
        _nvcc(srcs, LIBGSPN, ["-I" + os.path.join(ROOT, "include"), "-Xptxas", "-v"] if verbose else
              ["-I" + os.path.join(ROOT, "include")], verbose)
    return LIBGSPN


def build_synth(force: bool = False, verbose: bool = False) -> str:
    if force or _stale(LIBSYNTH, [SYNTH_SRC]):
        _nvcc([SYNTH_SRC], LIBSYNTH, None, verbose)
    return LIBSYNTH


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_gspn(force, verbose)
    build_synth(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
