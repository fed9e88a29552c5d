"""Host-side helpers for parity tests: seeded inputs regenerated on the host (synth, never copied from
the CUDA path), the oracle run on them, and the normwise error metric (R16)."""
from __future__ import annotations

import json
import os

import numpy as np

import synth
from synth.configs import Config

NAMES_W = ("w_l", "w_m", "w_r")
TOL = {"f32": 1e-5, "bf16": 2e-2}


def normwise(got: np.ndarray, ref: np.ndarray) -> float:
    """max |got - ref| / max |ref| (R16). 0 when both are identically zero."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    num = np.abs(got - ref).max() if ref.size else 0.0
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(num / den)


def record(test: str, name: str, err: float, tol: float) -> None:
    """Append one measured normwise error to $GSPN_ERRLOG (JSON lines; the GPU scripts set it to
    gpurun_out/parity_errors.jsonl, summarised under profiles/), so the margin to the tolerance is on record."""
    path = os.environ.get("GSPN_ERRLOG")
    if not path:
        return
    with open(path, "a") as f:
        f.write(json.dumps({"test": test, "tensor": name, "normwise": err, "tol": tol}) + "\n")


def check(test: str, name: str, got, ref, tol: float, per_slab: bool = True) -> float:
    """normwise(got, ref) <= tol per direction slab (5-D tensors) or whole; records and returns the max."""
    got, ref = np.asarray(got), np.asarray(ref)
    if per_slab and got.ndim == 5:
        errs = [normwise(got[k], ref[k]) for k in range(got.shape[0])]
    else:
        errs = [normwise(got, ref)]
    e = max(errs)
    record(test, name, e, tol)
    for k, ek in enumerate(errs):
        assert ek <= tol, f"{test}: {name}[slab {k}] normwise {ek:.3e} > {tol}"
    return e


def small_config(B, C, G, H, W, dirs, dtype, cfg_id=90) -> Config:
    return Config(f"t{B}x{C}x{G}x{H}x{W}d{dirs}{dtype}", cfg_id, B, C, G, H, W, dirs, dtype, "test shape")


def host_tensor(cfg: Config, name: str, shape, index_base=0, inner=None, outer_stride=None):
    """(io_values, float64) of a (slice of a) generated tensor."""
    v = synth.tensor(synth.seed_for(cfg.cfg_id), name, shape, cfg.dtype, index_base, inner, outer_stride)
    return v, synth.as_f64(v, cfg.dtype)


def host_inputs(cfg: Config):
    """Full host inputs of a small config: dict name -> (io_values, float64)."""
    D, B, C, G, H, W = cfg.D, cfg.B, cfg.C, cfg.G, cfg.H, cfg.W
    out = {"x": host_tensor(cfg, "x", (B, C, H, W))}
    for n in NAMES_W:
        out[n] = host_tensor(cfg, n, (D, B, G, H, W))
    out["lam"] = host_tensor(cfg, "lam", (D, B, C, H, W))
    out["dh"] = host_tensor(cfg, "dh", (D, B, C, H, W))
    return out


def unit_inputs(cfg: Config, b: int, g: int):
    """Host inputs of one unit (b, g) — all C/G channels, all directions — as a (B=1, C=Cg, G=1)
    problem, regenerated from the unsharded flat indices."""
    D, B, C, G, H, W = cfg.D, cfg.B, cfg.C, cfg.G, cfg.H, cfg.W
    HW, Cg = H * W, C // G
    u = b * G + g
    out = {"x": host_tensor(cfg, "x", (1, Cg, H, W), u * Cg * HW)}
    for n in NAMES_W:
        out[n] = host_tensor(cfg, n, (D, 1, 1, H, W), u * HW, HW, B * G * HW)
    out["lam"] = host_tensor(cfg, "lam", (D, 1, Cg, H, W), u * Cg * HW, Cg * HW, B * C * HW)
    out["dh"] = host_tensor(cfg, "dh", (D, 1, Cg, H, W), u * Cg * HW, Cg * HW, B * C * HW)
    return out


def round_io(a64: np.ndarray, dtype: str) -> np.ndarray:
    """Round float64 values to the I/O dtype (fp32 RN, then bf16 RNE), returned as float64."""
    a32 = np.asarray(a64, dtype=np.float64).astype(np.float32)
    if dtype == "bf16":
        return synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(a32)).astype(np.float64)
    return a32.astype(np.float64)


def to_torch(io_vals: np.ndarray, dtype: str, device):
    import torch

    if dtype == "bf16":
        t = torch.from_numpy(np.ascontiguousarray(io_vals).view(np.int16)).view(torch.bfloat16)
    else:
        t = torch.from_numpy(np.ascontiguousarray(io_vals, dtype=np.float32))
    return t.to(device)


def from_torch(t) -> np.ndarray:
    import torch

    return t.detach().to("cpu", torch.float64).numpy()


def io_from_f64(a64: np.ndarray, dtype: str) -> np.ndarray:
    """float64 values (already representable) -> I/O storage (fp32 array or bf16 bit patterns)."""
    a32 = np.asarray(a64).astype(np.float32)
    return synth.f32_to_bf16_bits(a32) if dtype == "bf16" else a32
