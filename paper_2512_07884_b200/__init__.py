"""B200-native GSPN / GSPN-2 line-scan propagation (arxiv 2512.07884).

Thin Python face of the C ABI in include/gspn.h: torch supplies device memory and the current
stream; every step of the scan runs in the CUDA kernels of libgspn.so. No CPU fallback exists.

  fwd(x, w_l, w_m, w_r, lam, dirs, groups, flags=0) -> h
  bwd(x, w_l, w_m, w_r, lam, h, dh, dirs, groups, flags=0) -> (dx, dw_l, dw_m, dw_r, dlam)

Shapes (gspn.h): x [B,C,H,W]; w_* [D,B,G,H,W]; lam, h, dh, dlam [D,B,C,H,W]; dx [B,C,H,W].
"""
from __future__ import annotations

import ctypes

from ._lib import GspnError, check, last_launch_count, last_path, lib  # noqa: F401

DIR_T2B, DIR_B2T, DIR_L2R, DIR_R2L, DIR_ALL = 0x1, 0x2, 0x4, 0x8, 0xF
FLAG_PRENORMALIZED = 0x1
FLAG_FORCE_GENERIC = 0x2
DTYPE_F32, DTYPE_BF16 = 0, 1


def _torch():
    import torch

    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return DTYPE_F32
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    raise TypeError(f"unsupported dtype {t.dtype} (float32 or bfloat16)")


def _check_tensors(named, dtype, device):
    for name, t in named:
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
        if t.device != device:
            raise ValueError(f"{name} is on {t.device}, expected {device}")
        if t.dtype != dtype:
            raise TypeError(f"{name} has dtype {t.dtype}, expected {dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")


def _stream_ptr(stream, device):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def popcount(d: int) -> int:
    return bin(int(d) & 0xF).count("1")


def fwd(x, w_l, w_m, w_r, lam, dirs: int = DIR_ALL, groups: int | None = None, flags: int = 0, out=None,
        stream=None):
    """Forward scan. groups defaults to C (per-channel weights)."""
    torch = _torch()
    B, C, H, W = x.shape
    G = C if groups is None else int(groups)
    D = popcount(dirs)
    if tuple(lam.shape) != (D, B, C, H, W):
        raise ValueError(f"lam shape {tuple(lam.shape)} != {(D, B, C, H, W)}")
    for n, w in (("w_l", w_l), ("w_m", w_m), ("w_r", w_r)):
        if tuple(w.shape) != (D, B, G, H, W):
            raise ValueError(f"{n} shape {tuple(w.shape)} != {(D, B, G, H, W)}")
    h = torch.empty_like(lam) if out is None else out
    _check_tensors([("x", x), ("w_l", w_l), ("w_m", w_m), ("w_r", w_r), ("lam", lam), ("h", h)], x.dtype, x.device)
    check(lib().gspn_fwd(x.data_ptr(), w_l.data_ptr(), w_m.data_ptr(), w_r.data_ptr(), lam.data_ptr(), h.data_ptr(),
                         B, C, H, W, dirs, G, _dtype_code(x), flags, _stream_ptr(stream, x.device)))
    return h


def workspace_bytes(B, C, H, W, dirs, groups, dtype_code) -> int:
    return int(lib().gspn_bwd_workspace_bytes(B, C, H, W, dirs, groups, dtype_code))


def algorithmic_bytes(B, C, H, W, dirs, groups, dtype_code, backward: bool) -> float:
    return float(lib().gspn_algorithmic_bytes(B, C, H, W, dirs, groups, dtype_code, int(backward)))


def bwd(x, w_l, w_m, w_r, lam, h, dh, dirs: int = DIR_ALL, groups: int | None = None, flags: int = 0,
        outs=None, workspace=None, stream=None):
    """Backward scan: returns (dx, dw_l, dw_m, dw_r, dlam)."""
    torch = _torch()
    B, C, H, W = x.shape
    G = C if groups is None else int(groups)
    dt = _dtype_code(x)
    if outs is None:
        outs = (torch.empty_like(x), torch.empty_like(w_l), torch.empty_like(w_m), torch.empty_like(w_r),
                torch.empty_like(lam))
    dx, dwl, dwm, dwr, dlam = outs
    _check_tensors([("x", x), ("w_l", w_l), ("w_m", w_m), ("w_r", w_r), ("lam", lam), ("h", h), ("dh", dh),
                    ("dx", dx), ("dw_l", dwl), ("dw_m", dwm), ("dw_r", dwr), ("dlam", dlam)], x.dtype, x.device)
    need = workspace_bytes(B, C, H, W, dirs, G, dt)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    check(lib().gspn_bwd(x.data_ptr(), w_l.data_ptr(), w_m.data_ptr(), w_r.data_ptr(), lam.data_ptr(), h.data_ptr(),
                         dh.data_ptr(), dx.data_ptr(), dwl.data_ptr(), dwm.data_ptr(), dwr.data_ptr(),
                         dlam.data_ptr(), B, C, H, W, dirs, G, dt, flags,
                         workspace.data_ptr() if need > 0 else None, workspace.numel(),
                         _stream_ptr(stream, x.device)))
    return dx, dwl, dwm, dwr, dlam
