"""ctypes loader for libgspn.so (the C ABI of include/gspn.h). Argument marshalling only.

The product path has NO CPU fallback: if the CUDA library is missing this raises immediately.
"""
from __future__ import annotations

import ctypes
import os

from .build import LIBGSPN

_lib = None

GSPN_OK = 0
STATUS = {0: "GSPN_OK", 1: "GSPN_ERR_INVALID_ARG", 2: "GSPN_ERR_UNSUPPORTED", 3: "GSPN_ERR_CUDA",
          4: "GSPN_ERR_INTERNAL"}


class GspnError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status
        self.detail = detail


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIBGSPN):
            raise ImportError(f"libgspn.so not built ({LIBGSPN}); run __graft_entry__.build() or "
                              "python -m paper_2512_07884_b200.build")
        path = LIBGSPN
        if os.environ.get("GSPN_EXPERIMENTS") and os.environ.get("GSPN_LIB"):  # A/B tooling only: another build
            path = os.environ["GSPN_LIB"]
        L = ctypes.CDLL(path)
        vp, i64, u32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
        L.gspn_fwd.argtypes = [vp] * 6 + [i64] * 4 + [u32, i64, ctypes.c_int, u32, vp]
        L.gspn_fwd.restype = ctypes.c_int
        L.gspn_bwd.argtypes = [vp] * 12 + [i64] * 4 + [u32, i64, ctypes.c_int, u32, vp, sz, vp]
        L.gspn_bwd.restype = ctypes.c_int
        # SURVEY §8(f) entry points (bound when present, so an older library still serves the core calls in
        # A/B timing runs; calling a missing one raises AttributeError)
        if hasattr(L, "gspn_fwd_local"):
            L.gspn_fwd_local.argtypes = [vp] * 6 + [i64] * 4 + [u32, i64, i64, ctypes.c_int, u32, vp]
            L.gspn_fwd_local.restype = ctypes.c_int
            L.gspn_bwd_local.argtypes = [vp] * 12 + [i64] * 4 + [u32, i64, i64, ctypes.c_int, u32, vp, sz, vp]
            L.gspn_bwd_local.restype = ctypes.c_int
        if hasattr(L, "gspn_fwd_ckpt"):
            L.gspn_fwd_ckpt.argtypes = [vp] * 7 + [i64] * 4 + [u32, i64, ctypes.c_int, u32, vp]
            L.gspn_fwd_ckpt.restype = ctypes.c_int
            L.gspn_bwd_recompute.argtypes = [vp] * 12 + [i64] * 4 + [u32, i64, ctypes.c_int, u32, vp, sz, vp]
            L.gspn_bwd_recompute.restype = ctypes.c_int
            for fn in ("gspn_ckpt_bytes", "gspn_bwd_recompute_workspace_bytes"):
                getattr(L, fn).argtypes = [i64] * 4 + [u32, i64, ctypes.c_int]
                getattr(L, fn).restype = sz
        if hasattr(L, "gspn_fwd_merged"):
            L.gspn_fwd_merged.argtypes = [vp] * 8 + [i64] * 4 + [u32, i64, ctypes.c_int, u32, vp, sz, vp]
            L.gspn_fwd_merged.restype = ctypes.c_int
            L.gspn_fwd_merged_workspace_bytes.argtypes = [i64] * 4 + [u32, i64, ctypes.c_int]
            L.gspn_fwd_merged_workspace_bytes.restype = sz
        if hasattr(L, "gspn_bwd_merged"):
            L.gspn_bwd_merged.argtypes = [vp] * 14 + [i64] * 4 + [u32, i64, ctypes.c_int, u32, vp, sz, vp]
            L.gspn_bwd_merged.restype = ctypes.c_int
            L.gspn_bwd_merged_workspace_bytes.argtypes = [i64] * 4 + [u32, i64, ctypes.c_int]
            L.gspn_bwd_merged_workspace_bytes.restype = sz
        L.gspn_bwd_workspace_bytes.argtypes = [i64] * 4 + [u32, i64, ctypes.c_int]
        L.gspn_bwd_workspace_bytes.restype = sz
        L.gspn_algorithmic_bytes.argtypes = [i64] * 4 + [u32, i64, ctypes.c_int, ctypes.c_int]
        L.gspn_algorithmic_bytes.restype = ctypes.c_double
        if hasattr(L, "gspn_merge_fwd"):
            L.gspn_merge_fwd.argtypes = [vp] * 3 + [i64] * 4 + [u32, ctypes.c_int, u32, vp]
            L.gspn_merge_fwd.restype = ctypes.c_int
            L.gspn_merge_bwd.argtypes = [vp] * 5 + [i64] * 4 + [u32, ctypes.c_int, u32, vp]
            L.gspn_merge_bwd.restype = ctypes.c_int
        if hasattr(L, "gspn_proxy_mix"):
            L.gspn_proxy_mix.argtypes = [vp] * 3 + [i64] * 5 + [ctypes.c_int, u32, vp]
            L.gspn_proxy_mix.restype = ctypes.c_int
            L.gspn_proxy_wgrad.argtypes = [vp] * 3 + [i64] * 5 + [ctypes.c_int, vp]
            L.gspn_proxy_wgrad.restype = ctypes.c_int
        L.gspn_status_string.argtypes = [ctypes.c_int]
        L.gspn_status_string.restype = ctypes.c_char_p
        L.gspn_last_error_detail.restype = ctypes.c_char_p
        L.gspn_last_path.restype = ctypes.c_char_p
        L.gspn_last_launch_count.restype = ctypes.c_int
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != GSPN_OK:
        raise GspnError(status, lib().gspn_last_error_detail().decode())


def last_path() -> str:
    return lib().gspn_last_path().decode()


def last_launch_count() -> int:
    return int(lib().gspn_last_launch_count())
