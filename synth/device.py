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


def index_maps(cfg: Config, sh: Shard) -> dict:
    """(index_base, inner, outer_stride) of every tensor of a shard: local flat index i maps to the
    unsharded flat index index_base + (i // inner) * outer_stride + i % inner (inner 0 = identity)."""
    HW = cfg.H * cfg.W
    Cg = cfg.C // cfg.G
    if sh.kind == "full":
        m = {n: (0, 0, 0) for n in ("x", "lam", "dh", "w_l", "w_m", "w_r")}
    elif sh.kind == "units":
        base = sh.unit0 * Cg * HW
        per_c = (base, sh.units * Cg * HW, cfg.B * cfg.C * HW)
        per_w = (sh.unit0 * HW, sh.units * HW, cfg.B * cfg.G * HW)
        m = {"x": (base, 0, 0), "lam": per_c, "dh": per_c, "w_l": per_w, "w_m": per_w, "w_r": per_w}
    else:  # channels [chan0, chan0 + chans) of the single unit; w replicated
        base = sh.chan0 * HW
        per_c = (base, sh.chans * HW, cfg.C * HW)
        m = {"x": (base, 0, 0), "lam": per_c, "dh": per_c, "w_l": (0, 0, 0), "w_m": (0, 0, 0), "w_r": (0, 0, 0)}
    return m


def shard_shapes(cfg: Config, sh: Shard) -> dict:
    D, H, W = cfg.D, cfg.H, cfg.W
    return {"x": (sh.B, sh.C, H, W), "lam": (D, sh.B, sh.C, H, W), "dh": (D, sh.B, sh.C, H, W),
            "w_l": (D, sh.B, sh.G, H, W), "w_m": (D, sh.B, sh.G, H, W), "w_r": (D, sh.B, sh.G, H, W)}


def full_shard(cfg: Config) -> Shard:
    return Shard(cfg.B, cfg.C, cfg.G, 0, cfg.B * cfg.G, 0, cfg.C, "full")


def host_shard_inputs(cfg: Config, sh: Shard | None = None) -> dict:
    """Host (numpy) twin of make_inputs: I/O-dtype values of every tensor of the shard."""
    from . import tensor

    sh = sh or full_shard(cfg)
    seed = seed_for(cfg.cfg_id)
    maps, shapes = index_maps(cfg, sh), shard_shapes(cfg, sh)
    out = {}
    for n, shape in shapes.items():
        base, inner, outer = maps[n]
        out[n] = tensor(seed, n, shape, cfg.dtype, base, inner or None, outer or None)
    return out


def make_inputs(cfg: Config, device, shard: Shard | None = None, with_dh: bool = True):
    """Allocate and fill x, w_l, w_m, w_r, lam (and dh) for (a shard of) config `cfg` on `device`."""
    import torch

    sh = shard or full_shard(cfg)
    seed = seed_for(cfg.cfg_id)
    dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    maps, shapes = index_maps(cfg, sh), shard_shapes(cfg, sh)
    out = {}
    for n, shape in shapes.items():
        if n == "dh" and not with_dh:
            out[n] = None
            continue
        t = torch.empty(shape, dtype=dt, device=device)
        base, inner, outer = maps[n]
        fill_(t, seed, n, base, inner, outer)
        out[n] = t
    return out
