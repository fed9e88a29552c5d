"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method: it only turns (seed, stream, flat index) into IEEE
values with a counter-based hash, so that the host (numpy, here) and the device (``libsynth.so``,
``synth/csrc/synth.cu``) produce bit-identical tensors, and any shard or any sampled plane can be
regenerated on its own from its flat index in the UNSHARDED tensor.

Recipe:
  key   = splitmix64((seed << 8) | stream)
  u     = (splitmix64(key ^ flat_index) >> 40) * 2**-24          (24 bits, exact in fp32/fp64)
  value = lo + (hi - lo) * u   in fp64, no contraction            (two IEEE roundings: mul, add)
        -> fp32 (round-to-nearest-even) -> bf16 (RNE) for bf16 tensors
Distributions mirror the paper's post-sigmoid affinities and gates and zero-mean
activations: x, dh ~ U[-1, 1); lam ~ U[0, 1); w_l, w_m, w_r ~ U[0.05, 1) (strictly positive, so the
row sum S > 0 everywhere and connectivity is dense); the merge's gate u ~ U[0, 1), dy, hs ~ U[-1, 1).
"""
from __future__ import annotations

import numpy as np

from .configs import CONFIGS, Config, get_config  # noqa: F401

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)

# tensor name -> (stream id, lo, hi)
STREAMS = {
    "x": (1, -1.0, 1.0),
    "w_l": (2, 0.05, 1.0),
    "w_m": (3, 0.05, 1.0),
    "w_r": (4, 0.05, 1.0),
    "lam": (5, 0.0, 1.0),
    "dh": (6, -1.0, 1.0),
    # SURVEY §8(f) NEXT-1 (output gate + merge): u is a post-sigmoid-like gate,
    # dy a zero-mean upstream gradient, hs a zero-mean stand-in state for merge-only tests
    "u": (7, 0.0, 1.0),
    "dy": (8, -1.0, 1.0),
    "hs": (9, -1.0, 1.0),
}


def seed_for(cfg_id: int) -> int:
    """seed = 7884 + 1000 * cfg."""
    return 7884 + 1000 * int(cfg_id)


def splitmix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
    return z ^ (z >> np.uint64(31))


def unit_u24(seed: int, stream: int, flat_index) -> np.ndarray:
    """u in [0, 1) with 24 random bits, as float64 (exact)."""
    key = splitmix64(np.uint64(((int(seed) << 8) | int(stream)) & 0xFFFFFFFFFFFFFFFF))
    idx = np.asarray(flat_index, dtype=np.uint64)
    bits = splitmix64(key ^ idx) >> np.uint64(40)
    return bits.astype(np.float64) * (1.0 / 16777216.0)


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 round-to-nearest-even, returned as uint16 bit patterns (finite inputs)."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    rounded = b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))
    return (rounded >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def values(seed: int, name: str, flat_index, dtype: str = "f32") -> np.ndarray:
    """Generated values at the given flat indices of tensor `name`.

    dtype "f32" -> float32 array; "bf16" -> uint16 array of bf16 bit patterns.
    """
    stream, lo, hi = STREAMS[name]
    u = unit_u24(seed, stream, flat_index)
    v64 = np.float64(lo) + np.float64(hi - lo) * u  # numpy: separate IEEE mul and add, no FMA
    v32 = v64.astype(np.float32)
    if dtype == "f32":
        return v32
    if dtype == "bf16":
        return f32_to_bf16_bits(v32)
    raise ValueError(f"unknown dtype {dtype!r}")


def as_f64(vals: np.ndarray, dtype: str) -> np.ndarray:
    """Exact float64 view of generated values (what the oracle consumes)."""
    if dtype == "bf16":
        return bf16_bits_to_f32(vals).astype(np.float64)
    return np.asarray(vals, dtype=np.float32).astype(np.float64)


def tensor(seed: int, name: str, shape, dtype: str = "f32", index_base: int = 0,
           inner: int | None = None, outer_stride: int | None = None) -> np.ndarray:
    """A whole (shard of a) tensor. Local flat index i maps to the unsharded flat index
    index_base + (i // inner) * outer_stride + (i % inner)  (identity when inner is None)."""
    n = int(np.prod(shape)) if len(shape) else 1
    i = np.arange(n, dtype=np.uint64)
    if inner is not None:
        g = np.uint64(index_base) + (i // np.uint64(inner)) * np.uint64(outer_stride) + (i % np.uint64(inner))
    else:
        g = i + np.uint64(index_base)
    return values(seed, name, g, dtype).reshape(shape)
