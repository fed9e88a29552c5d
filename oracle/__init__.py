"""fp64 CPU oracle of the GSPN line scan — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may
import this package. The product path (paper_2512_07884_b200) never imports, links or calls it.

The arithmetic lives in oracle/gspn_oracle.c (plain C loops, fp64, -ffp-contract=off); this module
only builds/loads it and marshals numpy float64 arrays. Layouts are those of include/gspn.h.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gspn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_gspn.so")
_lib = None

PRENORMALIZED = 1


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.gspn_oracle_fwd.argtypes = [d] * 6 + [i64] * 4 + [ctypes.c_uint, i64, ctypes.c_uint, i64, ctypes.c_int]
        lib.gspn_oracle_fwd.restype = ctypes.c_int
        lib.gspn_oracle_bwd.argtypes = [d] * 12 + [i64] * 4 + [ctypes.c_uint, i64, ctypes.c_uint, i64, ctypes.c_int]
        lib.gspn_oracle_bwd.restype = ctypes.c_int
        lib.gspn_oracle_detail.restype = ctypes.c_char_p
        lib.gspn_oracle_merge_fwd.argtypes = [d] * 3 + [i64, i64, ctypes.c_int]
        lib.gspn_oracle_merge_fwd.restype = None
        lib.gspn_oracle_merge_bwd.argtypes = [d] * 5 + [i64, i64, ctypes.c_int]
        lib.gspn_oracle_merge_bwd.restype = None
        lib.gspn_oracle_proxy_mix.argtypes = [d] * 3 + [i64] * 4
        lib.gspn_oracle_proxy_mix.restype = None
        lib.gspn_oracle_proxy_wgrad.argtypes = [d] * 3 + [i64] * 4
        lib.gspn_oracle_proxy_wgrad.restype = None
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    pass


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def fwd(x, wl, wm, wr, lam, dirs: int, groups: int, flags: int = 0, threads: int = 1, kchunk: int = 0) -> np.ndarray:
    """h [D,B,C,H,W] from x [B,C,H,W], w_* [D,B,G,H,W], lam [D,B,C,H,W] (float64).
    kchunk > 0: GSPN-local, h reset at every segment start."""
    x, wl, wm, wr, lam = map(_f64, (x, wl, wm, wr, lam))
    B, C, H, W = x.shape
    h = np.empty(lam.shape, dtype=np.float64)
    st = _load().gspn_oracle_fwd(_p(x), _p(wl), _p(wm), _p(wr), _p(lam), _p(h), B, C, H, W, dirs, groups,
                                 flags, kchunk, threads)
    if st:
        raise OracleError(f"oracle fwd status {st}: {_load().gspn_oracle_detail().decode()}")
    return h


def bwd(x, wl, wm, wr, lam, h, dh, dirs: int, groups: int, flags: int = 0, threads: int = 1, kchunk: int = 0):
    """(dx, dw_l, dw_m, dw_r, dlam) given saved h and upstream dh (float64)."""
    x, wl, wm, wr, lam, h, dh = map(_f64, (x, wl, wm, wr, lam, h, dh))
    B, C, H, W = x.shape
    dx = np.empty(x.shape)
    dwl, dwm, dwr = np.empty(wl.shape), np.empty(wl.shape), np.empty(wl.shape)
    dlam = np.empty(lam.shape)
    st = _load().gspn_oracle_bwd(_p(x), _p(wl), _p(wm), _p(wr), _p(lam), _p(h), _p(dh), _p(dx), _p(dwl), _p(dwm),
                                 _p(dwr), _p(dlam), B, C, H, W, dirs, groups, flags, kchunk, threads)
    if st:
        raise OracleError(f"oracle bwd status {st}: {_load().gspn_oracle_detail().decode()}")
    return dx, dwl, dwm, dwr, dlam


def merge_fwd(h, u, mean: bool = False) -> np.ndarray:
    """y [B,C,H,W] = s * sum_d u_d * h_d (Eq. 2, four passes combined; s = 1 or 1/D)."""
    h, u = _f64(h), _f64(u)
    D, N = h.shape[0], h[0].size
    y = np.empty(h.shape[1:])
    _load().gspn_oracle_merge_fwd(_p(h), _p(u), _p(y), D, N, int(mean))
    return y


def merge_bwd(h, u, dy, mean: bool = False):
    """(dh, du) [D,B,C,H,W] of merge_fwd given dy [B,C,H,W]."""
    h, u, dy = _f64(h), _f64(u), _f64(dy)
    D, N = h.shape[0], h[0].size
    dh, du = np.empty(h.shape), np.empty(h.shape)
    _load().gspn_oracle_merge_bwd(_p(h), _p(u), _p(dy), _p(dh), _p(du), D, N, int(mean))
    return dh, du


def proxy_mix(inp, M) -> np.ndarray:
    """out [B,Co,H,W] = sum_i M[o,i] inp[b,i] (1x1 projection); M [Co, Ci]."""
    inp, M = _f64(inp), _f64(M)
    B, Ci = inp.shape[:2]
    Co = M.shape[0]
    HW = int(np.prod(inp.shape[2:]))
    out = np.empty((B, Co) + inp.shape[2:])
    _load().gspn_oracle_proxy_mix(_p(inp), _p(M), _p(out), B, Ci, Co, HW)
    return out


def proxy_wgrad(dout, inp) -> np.ndarray:
    """dM [Co, Ci] = sum_{b,n} dout[b,o,n] inp[b,i,n] (weight gradient of proxy_mix)."""
    dout, inp = _f64(dout), _f64(inp)
    B, Co = dout.shape[:2]
    Ci = inp.shape[1]
    HW = int(np.prod(inp.shape[2:]))
    dM = np.empty((Co, Ci))
    _load().gspn_oracle_proxy_wgrad(_p(dout), _p(inp), _p(dM), B, Ci, Co, HW)
    return dM
