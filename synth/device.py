"""Device-side generation of the seeded inputs (libsynth.so), bit-identical to synth.values().

Shards: a rank that owns units [u0, u1) of the (b, g) unit space regenerates exactly
its slice of every tensor from the unsharded flat indices, presented to the scan as a problem with
B' = u1 - u0 units, C' = C/G channels and G' = 1 group. A channel split of one unit (config 5 at
N > 1) regenerates channels [c0, c1) of x / lam / dh and the whole (replicated) w.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

from . import STREAMS, seed_for
from .configs import Config

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB)
        L.synth_fill.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                 ctypes.c_void_p]
        L.synth_fill.restype = ctypes.c_int
        _lib = L
    return _lib


def fill_(t, seed: int, name: str, index_base: int = 0, inner: int = 0, outer_stride: int = 0, stream=None):
    import torch

    stream_id, lo, hi = STREAMS[name]
    dt = {torch.float32: 0, torch.bfloat16: 1}[t.dtype]
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    st = lib().synth_fill(t.data_ptr(), t.numel(), index_base, inner, outer_stride, seed, stream_id, lo, hi, dt,
                          ctypes.c_void_p(s.cuda_stream))
    if st != 0:
        raise RuntimeError(f"synth_fill failed with status {st}")
    return t


@dataclass
class Shard:
    """What one rank sees. (B, C, G) are the local problem dims passed to the ABI."""
    B: int
    C: int
    G: int
    unit0: int = 0
    units: int = 0
    chan0: int = 0
    chans: int = 0
    kind: str = "full"  # "full" | "units" | "channels"


def shard_for(cfg: Config, rank: int, world: int) -> Shard:
    """Contiguous equal split of the B*G units; a single-unit problem is split by channel instead."""
    U = cfg.B * cfg.G
    Cg = cfg.C // cfg.G
    if world == 1:
        return Shard(cfg.B, cfg.C, cfg.G, 0, U, 0, cfg.C, "full")
    if U >= world:
        u0 = rank * U // world
        u1 = (rank + 1) * U // world
        return Shard(u1 - u0, Cg, 1, u0, u1 - u0, 0, Cg, "units")
    if U == 1:
        c0 = rank * cfg.C // world
        c1 = (rank + 1) * cfg.C // world
        return Shard(1, c1 - c0, 1, 0, 1, c0, c1 - c0, "channels")
    raise ValueError(f"cannot shard {U} units over {world} ranks")


def make_inputs(cfg: Config, device, shard: Shard | None = None, with_dh: bool = True):
    """Allocate and fill x, w_l, w_m, w_r, lam (and dh) for (a shard of) config `cfg` on `device`."""
    import torch

    sh = shard or Shard(cfg.B, cfg.C, cfg.G, 0, cfg.B * cfg.G, 0, cfg.C, "full")
    seed = seed_for(cfg.cfg_id)
    dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    D, H, W = cfg.D, cfg.H, cfg.W
    HW = H * W
    Cg = cfg.C // cfg.G
    out = {}
    x = torch.empty((sh.B, sh.C, H, W), dtype=dt, device=device)
    lam = torch.empty((D, sh.B, sh.C, H, W), dtype=dt, device=device)
    ws = [torch.empty((D, sh.B, sh.G, H, W), dtype=dt, device=device) for _ in range(3)]
    dh = torch.empty((D, sh.B, sh.C, H, W), dtype=dt, device=device) if with_dh else None
    if sh.kind == "full":
        fill_(x, seed, "x")
        fill_(lam, seed, "lam")
        for w, n in zip(ws, ("w_l", "w_m", "w_r")):
            fill_(w, seed, n)
        if dh is not None:
            fill_(dh, seed, "dh")
    elif sh.kind == "units":
        base = sh.unit0 * Cg * HW
        fill_(x, seed, "x", base)
        fill_(lam, seed, "lam", base, sh.units * Cg * HW, cfg.B * cfg.C * HW)
        for w, n in zip(ws, ("w_l", "w_m", "w_r")):
            fill_(w, seed, n, sh.unit0 * HW, sh.units * HW, cfg.B * cfg.G * HW)
        if dh is not None:
            fill_(dh, seed, "dh", base, sh.units * Cg * HW, cfg.B * cfg.C * HW)
    else:  # channels of the single unit
        base = sh.chan0 * HW
        fill_(x, seed, "x", base)
        fill_(lam, seed, "lam", base, sh.chans * HW, cfg.C * HW)
        for w, n in zip(ws, ("w_l", "w_m", "w_r")):
            fill_(w, seed, n)
        if dh is not None:
            fill_(dh, seed, "dh", base, sh.chans * HW, cfg.C * HW)
    out["x"], out["lam"], out["w_l"], out["w_m"], out["w_r"], out["dh"] = x, lam, ws[0], ws[1], ws[2], dh
    return out
