"""Build the in-tree native libraries with nvcc for sm_100a (no JIT cache; the .so files travel with
the repo snapshot to the GPU box).

  paper_2512_07884_b200/lib/libgspn.so   the C ABI of include/gspn.h (all CUDA kernels)
  synth/libsynth.so                      the device twin of the seeded input generator
"""
from __future__ import annotations

import glob
import hashlib
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


def _digest(sources: list[str], flags: list[str]) -> str:
    """Content hash of every source/header and the compile flags: a library is reused only if it was built
    from exactly these bytes (an mtime test would trust a copied-in or interrupted-A/B library)."""
    h = hashlib.sha256()
    for f in [*ARCH, *COMMON, *flags]:
        h.update(f.encode() + b"\0")
    for s in sorted(sources):
        h.update(os.path.relpath(s, ROOT).encode() + b"\0")
        with open(s, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def _stale(target: str, sources: list[str], flags: list[str] | None = None) -> bool:
    if not os.path.exists(target) or not os.path.exists(target + ".hash"):
        return True
    with open(target + ".hash") as fh:
        return fh.read().strip() != _digest(sources, flags or [])


def _nvcc(sources: list[str], out: str, extra: list[str] | None = None, verbose: bool = False,
          deps: list[str] | None = None) -> None:
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + f".tmp{os.getpid()}"
    if len(sources) == 1:
        cmd = [NVCC, *ARCH, *COMMON, *(extra or []), "-o", tmp, *sources]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    else:  # one object per translation unit, compiled in parallel, then one shared link
        from concurrent.futures import ThreadPoolExecutor

        objdir = os.path.join(os.path.dirname(out), f".obj{os.getpid()}")
        os.makedirs(objdir, exist_ok=True)
        flags = [f for f in COMMON if f != "-shared"]
        objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in sources]

        def cc(pair):
            src, obj = pair
            cmd = [NVCC, *ARCH, *flags, *(extra or []), "-c", "-o", obj, src]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)

        with ThreadPoolExecutor(max_workers=max(1, min(len(sources), os.cpu_count() or 1))) as ex:
            list(ex.map(cc, zip(sources, objs)))
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs])
        for o in objs:
            os.remove(o)
        os.rmdir(objdir)
    os.replace(tmp, out)
    with open(out + ".hash", "w") as fh:
        fh.write(_digest(deps or sources, [f for f in (extra or []) if f not in ("-Xptxas", "-v")]))


def build_gspn(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(glob.glob(os.path.join(CSRC, "*.h"))) + \
        [os.path.join(ROOT, "include", "gspn.h")]
    inc = ["-I" + os.path.join(ROOT, "include")]
    if force or _stale(LIBGSPN, deps, inc):
        _nvcc(srcs, LIBGSPN, inc + (["-Xptxas", "-v"] if verbose else []), verbose, deps)
    return LIBGSPN


def build_synth(force: bool = False, verbose: bool = False) -> str:
    if force or _stale(LIBSYNTH, [SYNTH_SRC]):
        _nvcc([SYNTH_SRC], LIBSYNTH, None, verbose, [SYNTH_SRC])
    return LIBSYNTH


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_gspn(force, verbose)
    build_synth(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
