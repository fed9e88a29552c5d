"""B200-native GSPN / GSPN-2 line-scan propagation (arxiv 2512.07884).

Thin Python face of the C ABI in include/gspn.h: torch supplies device memory and the current
stream; every step of the scan runs in the CUDA kernels of libgspn.so. No CPU fallback exists.

  fwd(x, w_l, w_m, w_r, lam, dirs, groups, flags=0) -> h
  bwd(x, w_l, w_m, w_r, lam, h, dh, dirs, groups, flags=0) -> (dx, dw_l, dw_m, dw_r, dlam)
  fwd(..., kchunk=k) / bwd(..., kchunk=k)                (GSPN-local)
  merge_fwd(h, u, dirs, mean=False) -> y               (output gate + direction merge, Eq. 2)
  merge_bwd(h, u, dy, dirs, mean=False) -> (dh, du)
  proxy_mix(inp, M, transpose=False) -> out             (1x1 proxy projection)
  proxy_wgrad(dout, inp) -> dM (fp32)

Shapes (gspn.h): x [B,C,H,W]; w_* [D,B,G,H,W]; lam, h, dh, dlam [D,B,C,H,W]; dx [B,C,H,W].
"""
from __future__ import annotations

import ctypes

from ._lib import GspnError, check, last_launch_count, last_path, lib  # noqa: F401

DIR_T2B, DIR_B2T, DIR_L2R, DIR_R2L, DIR_ALL = 0x1, 0x2, 0x4, 0x8, 0xF
FLAG_PRENORMALIZED = 0x1
FLAG_FORCE_GENERIC = 0x2
FLAG_MERGE_MEAN = 0x4
FLAG_PROXY_TRANSPOSE = 0x8
FLAG_FORCE_SPLIT = 0x10
FLAG_DW_F32 = 0x20
FLAG_PROXY_SIMT = 0x10  # proxy_mix only
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


def _check_shapes(named):
    """named: (name, tensor, expected shape). The C ABI sees only pointers, so a mis-shaped tensor would
    become an out-of-bounds device access: every tensor the call reads or writes is checked here."""
    for name, t, shape in named:
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} shape {tuple(t.shape)} != expected {tuple(shape)}")


def _scan_shapes(x, dirs, G):
    """(B, C, H, W, D) and the expected shapes of x, w_*, lam-like tensors (gspn.h layouts)."""
    if x.dim() != 4:
        raise ValueError(f"x must be [B, C, H, W], got {tuple(x.shape)}")
    B, C, H, W = x.shape
    D = popcount(dirs)
    return (B, C, H, W, D), (B, C, H, W), (D, B, G, H, W), (D, B, C, H, W)


def fwd(x, w_l, w_m, w_r, lam, dirs: int = DIR_ALL, groups: int | None = None, flags: int = 0, out=None,
        stream=None, kchunk: int = 0):
    """Forward scan. groups defaults to C (per-channel weights); kchunk > 0: GSPN-local (gspn_fwd_local)."""
    torch = _torch()
    G = x.shape[1] if groups is None else int(groups)
    (B, C, H, W, D), sx, sw, sl = _scan_shapes(x, dirs, G)
    h = torch.empty_like(lam) if out is None else out
    _check_shapes([("lam", lam, sl), ("w_l", w_l, sw), ("w_m", w_m, sw), ("w_r", w_r, sw), ("h (out)", h, sl)])
    _check_tensors([("x", x), ("w_l", w_l), ("w_m", w_m), ("w_r", w_r), ("lam", lam), ("h", h)], x.dtype, x.device)
    ptrs = (x.data_ptr(), w_l.data_ptr(), w_m.data_ptr(), w_r.data_ptr(), lam.data_ptr(), h.data_ptr())
    if kchunk:
        check(lib().gspn_fwd_local(*ptrs, B, C, H, W, dirs, G, int(kchunk), _dtype_code(x), flags,
                                   _stream_ptr(stream, x.device)))
    else:
        check(lib().gspn_fwd(*ptrs, B, C, H, W, dirs, G, _dtype_code(x), flags, _stream_ptr(stream, x.device)))
    return h


def workspace_bytes(B, C, H, W, dirs, groups, dtype_code) -> int:
    return int(lib().gspn_bwd_workspace_bytes(B, C, H, W, dirs, groups, dtype_code))


def algorithmic_bytes(B, C, H, W, dirs, groups, dtype_code, backward: bool) -> float:
    return float(lib().gspn_algorithmic_bytes(B, C, H, W, dirs, groups, dtype_code, int(backward)))


def bwd(x, w_l, w_m, w_r, lam, h, dh, dirs: int = DIR_ALL, groups: int | None = None, flags: int = 0,
        outs=None, workspace=None, stream=None, kchunk: int = 0):
    """Backward scan: returns (dx, dw_l, dw_m, dw_r, dlam)."""
    torch = _torch()
    G = x.shape[1] if groups is None else int(groups)
    (B, C, H, W, D), sx, sw, sl = _scan_shapes(x, dirs, G)
    dt = _dtype_code(x)
    dw_dtype = torch.float32 if flags & FLAG_DW_F32 else x.dtype  # fp32 partial dw (cross-device reduction)
    if outs is None:
        outs = (torch.empty_like(x), torch.empty_like(w_l, dtype=dw_dtype), torch.empty_like(w_m, dtype=dw_dtype),
                torch.empty_like(w_r, dtype=dw_dtype), torch.empty_like(lam))
    if len(outs) != 5:
        raise ValueError("outs must be (dx, dw_l, dw_m, dw_r, dlam)")
    dx, dwl, dwm, dwr, dlam = outs
    _check_shapes([("w_l", w_l, sw), ("w_m", w_m, sw), ("w_r", w_r, sw), ("lam", lam, sl), ("h", h, sl),
                   ("dh", dh, sl), ("dx (out)", dx, sx), ("dw_l (out)", dwl, sw), ("dw_m (out)", dwm, sw),
                   ("dw_r (out)", dwr, sw), ("dlam (out)", dlam, sl)])
    _check_tensors([("x", x), ("w_l", w_l), ("w_m", w_m), ("w_r", w_r), ("lam", lam), ("h", h), ("dh", dh),
                    ("dx", dx), ("dlam", dlam)], x.dtype, x.device)
    _check_tensors([("dw_l", dwl), ("dw_m", dwm), ("dw_r", dwr)], dw_dtype, x.device)
    need = workspace_bytes(B, C, H, W, dirs, G, dt)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    ptrs = (x.data_ptr(), w_l.data_ptr(), w_m.data_ptr(), w_r.data_ptr(), lam.data_ptr(), h.data_ptr(),
            dh.data_ptr(), dx.data_ptr(), dwl.data_ptr(), dwm.data_ptr(), dwr.data_ptr(), dlam.data_ptr())
    ws = (workspace.data_ptr() if need > 0 else None, workspace.numel(), _stream_ptr(stream, x.device))
    if kchunk:
        check(lib().gspn_bwd_local(*ptrs, B, C, H, W, dirs, G, int(kchunk), dt, flags, *ws))
    else:
        check(lib().gspn_bwd(*ptrs, B, C, H, W, dirs, G, dt, flags, *ws))
    return dx, dwl, dwm, dwr, dlam


def merge_fwd(h, u, dirs: int = DIR_ALL, mean: bool = False, out=None, stream=None):
    """y [B,C,H,W] = s * sum_d u_d * h_d (s = 1, or 1/D with mean=True)."""
    torch = _torch()
    D, B, C, H, W = h.shape
    if D != popcount(dirs) or tuple(u.shape) != tuple(h.shape):
        raise ValueError(f"h {tuple(h.shape)} / u {tuple(u.shape)} do not match dirs=0x{dirs:x}")
    y = torch.empty(h.shape[1:], dtype=h.dtype, device=h.device) if out is None else out
    _check_shapes([("y (out)", y, h.shape[1:])])
    _check_tensors([("h", h), ("u", u), ("y", y)], h.dtype, h.device)
    check(lib().gspn_merge_fwd(h.data_ptr(), u.data_ptr(), y.data_ptr(), B, C, H, W, dirs, _dtype_code(h),
                               FLAG_MERGE_MEAN if mean else 0, _stream_ptr(stream, h.device)))
    return y


def merge_bwd(h, u, dy, dirs: int = DIR_ALL, mean: bool = False, outs=None, stream=None):
    """(dh, du) [D,B,C,H,W] of merge_fwd given dy [B,C,H,W]."""
    torch = _torch()
    D, B, C, H, W = h.shape
    if D != popcount(dirs) or tuple(u.shape) != tuple(h.shape) or tuple(dy.shape) != tuple(h.shape[1:]):
        raise ValueError("h / u / dy shapes do not match")
    dh, du = (torch.empty_like(h), torch.empty_like(h)) if outs is None else outs
    _check_shapes([("dh (out)", dh, h.shape), ("du (out)", du, h.shape)])
    _check_tensors([("h", h), ("u", u), ("dy", dy), ("dh", dh), ("du", du)], h.dtype, h.device)
    check(lib().gspn_merge_bwd(h.data_ptr(), u.data_ptr(), dy.data_ptr(), dh.data_ptr(), du.data_ptr(), B, C, H, W,
                               dirs, _dtype_code(h), FLAG_MERGE_MEAN if mean else 0, _stream_ptr(stream, h.device)))
    return dh, du


def fwd_ckpt(x, w_l, w_m, w_r, lam, dirs: int = DIR_ALL, groups: int | None = None, flags: int = 0,
             keep_h: bool = False, ckpt=None, h_out=None, stream=None):
    """Forward with fp32 checkpoints for the recompute backward (gspn_fwd_ckpt, NEXT-3): returns (ckpt, h),
    h None unless keep_h."""
    torch = _torch()
    G = x.shape[1] if groups is None else int(groups)
    (B, C, H, W, D), sx, sw, sl = _scan_shapes(x, dirs, G)
    dt = _dtype_code(x)
    nb = int(lib().gspn_ckpt_bytes(B, C, H, W, dirs, G, dt))
    if ckpt is None or ckpt.numel() * 4 < nb:
        ckpt = torch.empty(max(nb // 4, 4), dtype=torch.float32, device=x.device)
    h = (torch.empty_like(lam) if h_out is None else h_out) if keep_h else None
    named = [("lam", lam, sl), ("w_l", w_l, sw), ("w_m", w_m, sw), ("w_r", w_r, sw)]
    if h is not None:
        named.append(("h (out)", h, sl))
    _check_shapes(named)
    _check_tensors([(n, t) for n, t, _ in named] + [("x", x)], x.dtype, x.device)
    _check_tensors([("ckpt", ckpt)], torch.float32, x.device)
    check(lib().gspn_fwd_ckpt(x.data_ptr(), w_l.data_ptr(), w_m.data_ptr(), w_r.data_ptr(), lam.data_ptr(),
                              h.data_ptr() if h is not None else None, ckpt.data_ptr(), B, C, H, W, dirs, G, dt, flags,
                              _stream_ptr(stream, x.device)))
    return ckpt, h


def bwd_recompute(x, w_l, w_m, w_r, lam, ckpt, dh, dirs: int = DIR_ALL, groups: int | None = None, flags: int = 0,
                  outs=None, workspace=None, stream=None):
    """Backward from checkpoints instead of h (gspn_bwd_recompute, NEXT-3): returns (dx, dw_l, dw_m, dw_r, dlam)."""
    torch = _torch()
    G = x.shape[1] if groups is None else int(groups)
    (B, C, H, W, D), sx, sw, sl = _scan_shapes(x, dirs, G)
    dt = _dtype_code(x)
    if outs is None:
        outs = (torch.empty_like(x), torch.empty_like(w_l), torch.empty_like(w_m), torch.empty_like(w_r),
                torch.empty_like(lam))
    dx, dwl, dwm, dwr, dlam = outs
    _check_shapes([("w_l", w_l, sw), ("w_m", w_m, sw), ("w_r", w_r, sw), ("lam", lam, sl), ("dh", dh, sl),
                   ("dx (out)", dx, sx), ("dw_l (out)", dwl, sw), ("dw_m (out)", dwm, sw), ("dw_r (out)", dwr, sw),
                   ("dlam (out)", dlam, sl)])
    _check_tensors([("x", x), ("w_l", w_l), ("w_m", w_m), ("w_r", w_r), ("lam", lam), ("dh", dh), ("dx", dx),
                    ("dw_l", dwl), ("dw_m", dwm), ("dw_r", dwr), ("dlam", dlam)], x.dtype, x.device)
    _check_tensors([("ckpt", ckpt)], torch.float32, x.device)
    if ckpt.numel() * 4 < int(lib().gspn_ckpt_bytes(B, C, H, W, dirs, G, dt)):
        raise ValueError("ckpt smaller than gspn_ckpt_bytes")
    need = int(lib().gspn_bwd_recompute_workspace_bytes(B, C, H, W, dirs, G, dt))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    check(lib().gspn_bwd_recompute(x.data_ptr(), w_l.data_ptr(), w_m.data_ptr(), w_r.data_ptr(), lam.data_ptr(),
                                   ckpt.data_ptr(), dh.data_ptr(), dx.data_ptr(), dwl.data_ptr(), dwm.data_ptr(),
                                   dwr.data_ptr(), dlam.data_ptr(), B, C, H, W, dirs, G, dt, flags,
                                   workspace.data_ptr(), workspace.numel(), _stream_ptr(stream, x.device)))
    return dx, dwl, dwm, dwr, dlam


def fwd_merged(x, w_l, w_m, w_r, lam, u, dirs: int = DIR_ALL, groups: int | None = None, mean: bool = False,
               flags: int = 0, keep_h: bool = True, out=None, h_out=None, workspace=None, stream=None):
    """Forward scan + output gate + direction merge (gspn_fwd_merged, NEXT-1): returns (y, h), h None when
    keep_h is False (then h lives in a scratch workspace)."""
    torch = _torch()
    G = x.shape[1] if groups is None else int(groups)
    (B, C, H, W, D), sx, sw, sl = _scan_shapes(x, dirs, G)
    dt = _dtype_code(x)
    y = torch.empty_like(x) if out is None else out
    h = (torch.empty_like(lam) if h_out is None else h_out) if keep_h else None
    named = [("lam", lam, sl), ("u", u, sl), ("w_l", w_l, sw), ("w_m", w_m, sw), ("w_r", w_r, sw), ("y (out)", y, sx)]
    if h is not None:
        named.append(("h (out)", h, sl))
    _check_shapes(named)
    _check_tensors([(n, t) for n, t, _ in named] + [("x", x)], x.dtype, x.device)
    ws_ptr, ws_n = None, 0
    if h is None:
        need = int(lib().gspn_fwd_merged_workspace_bytes(B, C, H, W, dirs, G, dt))
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
        ws_ptr, ws_n = workspace.data_ptr(), workspace.numel()
    check(lib().gspn_fwd_merged(x.data_ptr(), w_l.data_ptr(), w_m.data_ptr(), w_r.data_ptr(), lam.data_ptr(),
                                u.data_ptr(), h.data_ptr() if h is not None else None, y.data_ptr(), B, C, H, W, dirs, G,
                                dt, flags | (FLAG_MERGE_MEAN if mean else 0), ws_ptr, ws_n,
                                _stream_ptr(stream, x.device)))
    return y, h


def bwd_merged(x, w_l, w_m, w_r, lam, h, u, dy, dirs: int = DIR_ALL, groups: int | None = None, mean: bool = False,
               flags: int = 0, outs=None, workspace=None, stream=None):
    """Backward through the scan and the output gate + direction merge (gspn_bwd_merged, NEXT-1):
    returns (dx, dw_l, dw_m, dw_r, dlam, du)."""
    torch = _torch()
    G = x.shape[1] if groups is None else int(groups)
    (B, C, H, W, D), sx, sw, sl = _scan_shapes(x, dirs, G)
    dt = _dtype_code(x)
    if outs is None:
        outs = (torch.empty_like(x), torch.empty_like(w_l), torch.empty_like(w_m), torch.empty_like(w_r),
                torch.empty_like(lam), torch.empty_like(lam))
    if len(outs) != 6:
        raise ValueError("outs must be (dx, dw_l, dw_m, dw_r, dlam, du)")
    dx, dwl, dwm, dwr, dlam, du = outs
    _check_shapes([("w_l", w_l, sw), ("w_m", w_m, sw), ("w_r", w_r, sw), ("lam", lam, sl), ("h", h, sl),
                   ("u", u, sl), ("dy", dy, sx), ("dx (out)", dx, sx), ("dw_l (out)", dwl, sw),
                   ("dw_m (out)", dwm, sw), ("dw_r (out)", dwr, sw), ("dlam (out)", dlam, sl), ("du (out)", du, sl)])
    _check_tensors([("x", x), ("w_l", w_l), ("w_m", w_m), ("w_r", w_r), ("lam", lam), ("h", h), ("u", u), ("dy", dy),
                    ("dx", dx), ("dw_l", dwl), ("dw_m", dwm), ("dw_r", dwr), ("dlam", dlam), ("du", du)],
                   x.dtype, x.device)
    need = int(lib().gspn_bwd_merged_workspace_bytes(B, C, H, W, dirs, G, dt))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    check(lib().gspn_bwd_merged(x.data_ptr(), w_l.data_ptr(), w_m.data_ptr(), w_r.data_ptr(), lam.data_ptr(),
                                h.data_ptr(), u.data_ptr(), dy.data_ptr(), dx.data_ptr(), dwl.data_ptr(),
                                dwm.data_ptr(), dwr.data_ptr(), dlam.data_ptr(), du.data_ptr(), B, C, H, W, dirs, G, dt,
                                flags | (FLAG_MERGE_MEAN if mean else 0), workspace.data_ptr(), workspace.numel(),
                                _stream_ptr(stream, x.device)))
    return dx, dwl, dwm, dwr, dlam, du


def proxy_mix(inp, M, transpose: bool = False, out=None, stream=None, simt: bool = False):
    """out [B,Co,H,W] = sum_i M[o,i] inp[b,i]; M [Co, Ci] (or [Ci, Co] used transposed). bf16 shapes the
    tensor-core kernel tiles run on tcgen05 unless simt=True (testing)."""
    torch = _torch()
    B, Ci, H, W = inp.shape
    if transpose:
        if M.shape[0] != Ci:
            raise ValueError(f"M {tuple(M.shape)} (transposed) does not match Ci={Ci}")
        Co = M.shape[1]
    else:
        if M.shape[1] != Ci:
            raise ValueError(f"M {tuple(M.shape)} does not match Ci={Ci}")
        Co = M.shape[0]
    out = torch.empty((B, Co, H, W), dtype=inp.dtype, device=inp.device) if out is None else out
    _check_shapes([("M", M, (Ci, Co) if transpose else (Co, Ci)), ("out", out, (B, Co, H, W))])
    _check_tensors([("in", inp), ("M", M), ("out", out)], inp.dtype, inp.device)
    check(lib().gspn_proxy_mix(inp.data_ptr(), M.data_ptr(), out.data_ptr(), B, Ci, Co, H, W, _dtype_code(inp),
                               (FLAG_PROXY_TRANSPOSE if transpose else 0) | (FLAG_PROXY_SIMT if simt else 0),
                               _stream_ptr(stream, inp.device)))
    return out


def proxy_wgrad(dout, inp, out=None, stream=None):
    """dM [Co, Ci] (float32) = sum_{b,pixels} dout[b,o] . inp[b,i]."""
    torch = _torch()
    B, Co, H, W = dout.shape
    Ci = inp.shape[1]
    dM = torch.empty((Co, Ci), dtype=torch.float32, device=dout.device) if out is None else out
    if inp.dim() != 4:
        raise ValueError(f"in must be [B, Ci, H, W], got {tuple(inp.shape)}")
    _check_shapes([("in", inp, (B, Ci, H, W)), ("dM (out)", dM, (Co, Ci))])
    _check_tensors([("dout", dout), ("in", inp)], dout.dtype, dout.device)
    _check_tensors([("dM", dM)], torch.float32, dout.device)
    check(lib().gspn_proxy_wgrad(dout.data_ptr(), inp.data_ptr(), dM.data_ptr(), B, Ci, Co, H, W, _dtype_code(dout),
                                 _stream_ptr(stream, dout.device)))
    return dM
