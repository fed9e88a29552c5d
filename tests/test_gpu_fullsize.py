"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times (device-generated
inputs, one fwd and one bwd call through the C ABI, the bwd consuming the GPU's own h).

The oracle recomputes sampled units (b, g) — all their channels and directions — from host-regenerated
inputs (synth, flat indices of the unsharded tensors), and the device generator is checked bit-exact
against the host generator on the same samples. Whole-tensor properties that hold at any size
(adjoint dot test, Euler identity of the normalisation) cover everything the samples do not.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2512_07884_b200 as gspn
import synth
from synth.configs import get_config
from synth.device import make_inputs
from tests.parity_utils import TOL, check, from_torch, normwise, record, unit_inputs

pytestmark = pytest.mark.gpu
NTHREADS = oracle.default_threads()


def _run(cfg, device, kchunk=0):
    t = make_inputs(cfg, device)
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], cfg.dirs, cfg.G, kchunk=kchunk)
    g = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], cfg.dirs, cfg.G, kchunk=kchunk)
    return t, h, g


def _sample_units(cfg, n):
    U = cfg.B * cfg.G
    picks = {0, U - 1}
    rng = np.random.default_rng(cfg.cfg_id)
    while len(picks) < min(n, U):
        picks.add(int(rng.integers(0, U)))
    return sorted(picks)


def _check_unit(cfg, t, h, grads, u, kchunk=0):
    b, g = divmod(u, cfg.G)
    Cg = cfg.C // cfg.G
    c0 = g * Cg
    inp = unit_inputs(cfg, b, g)
    # the device generator reproduces the host generator bit for bit on this unit
    x_dev = t["x"][b, c0:c0 + Cg].contiguous().cpu()
    x_host = inp["x"][0][0]
    if cfg.dtype == "bf16":
        assert np.array_equal(x_dev.view(dtype=__import__("torch").int16).numpy().view(np.uint16), x_host)
    else:
        assert np.array_equal(x_dev.numpy(), x_host)
    f = {k: v[1] for k, v in inp.items()}
    h_ref = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], cfg.dirs, 1, threads=1, kchunk=kchunk)
    gr = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], h_ref, f["dh"], cfg.dirs, 1, threads=1,
                    kchunk=kchunk)
    tol = TOL[cfg.dtype]
    import os

    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0] + f"[unit {u}]"
    check(test, "h", from_torch(h[:, b:b + 1, c0:c0 + Cg]), h_ref, tol)
    got = [from_torch(grads[0][b:b + 1, c0:c0 + Cg])] + \
          [from_torch(grads[i][:, b:b + 1, g:g + 1]) for i in (1, 2, 3)] + \
          [from_torch(grads[4][:, b:b + 1, c0:c0 + Cg])]
    for name, a, r in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), got, gr):
        check(test, name, a, r, tol)


def _dot(a, b):
    import torch

    return float(torch.sum(a.to(torch.float64) * b.to(torch.float64)))


def _check_identities(cfg, t, h, grads):
    """<dh, h> = <dx, x> = sum_d <dlam_d, lam_d>; w_l dw_l + w_m dw_m + w_r dw_r = 0 per pixel."""
    import torch

    dx, dwl, dwm, dwr, dlam = grads
    a = _dot(t["dh"], h)
    bx = _dot(dx, t["x"])
    bl = _dot(dlam, t["lam"])
    scale = float(torch.sum(torch.abs(t["dh"].to(torch.float64) * h.to(torch.float64))))
    tol = 1e-4 if cfg.dtype == "f32" else 2e-2
    assert abs(bx - a) <= tol * scale, (a, bx)
    assert abs(bl - a) <= tol * scale, (a, bl)
    f = lambda v: v.to(torch.float32)
    e = f(t["w_l"]) * f(dwl) + f(t["w_m"]) * f(dwm) + f(t["w_r"]) * f(dwr)
    mag = torch.maximum(torch.maximum((f(t["w_l"]) * f(dwl)).abs(), (f(t["w_m"]) * f(dwm)).abs()),
                        (f(t["w_r"]) * f(dwr)).abs())
    assert float(e.abs().max()) <= 4 * tol * float(mag.max())


@pytest.mark.parametrize("name,nunits,dtype", [("1", 8, None), ("2", 4, None), ("3a", 64, None), ("3a", 64, "f32"),
                                               ("3b", 3, None), ("4", 3, None)])
def test_config_sampled_parity(name, nunits, dtype, cuda_device):
    """dtype None: the config's own I/O dtype; "f32": the fp32 parity run SURVEY §8 asks for (3a)."""
    cfg = get_config(name)
    if dtype:
        cfg = cfg.with_(dtype=dtype)
    t, h, grads = _run(cfg, cuda_device)
    for u in _sample_units(cfg, nunits):
        _check_unit(cfg, t, h, grads, u)
    _check_identities(cfg, t, h, grads)


@pytest.mark.parametrize("name,nunits,kchunk", [("2", 3, 14), ("3b", 2, 7), ("4", 2, 128)])
def test_config_sampled_parity_local(name, nunits, kchunk, cuda_device):
    """GSPN-local at full size in the bench's launch configuration (bench `next.local`)."""
    cfg = get_config(name)
    t, h, grads = _run(cfg, cuda_device, kchunk)
    for u in _sample_units(cfg, nunits):
        _check_unit(cfg, t, h, grads, u, kchunk)
    _check_identities(cfg, t, h, grads)


@pytest.mark.slow
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_config5_parity(dtype, cuda_device):
    """Config 5: one unit of 40 channels over 2048^2 (L = P = 2048), bf16 and the fp32 parity run. h, dx,
    dlam on sampled channels from per-channel oracle runs; dw (summed over all 40 channels) from the sum
    of per-channel oracle runs, which equals the grouped result because the normalisation Jacobian is
    linear in the tap gradients (tests/test_oracle.py::test_grouped_dw_is_channel_sum_of_per_channel).
    The oracle runs on the UNROUNDED fp64 h (end to end); the measured margins go to $GSPN_ERRLOG."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    cfg = get_config("5").with_(dtype=dtype)
    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    t, h, grads = _run(cfg, cuda_device)
    _check_identities(cfg, t, h, grads)
    HW = cfg.H * cfg.W
    seed = synth.seed_for(cfg.cfg_id)
    D = cfg.D

    def w_planes():
        out = {}
        for n in ("w_l", "w_m", "w_r"):
            v = synth.tensor(seed, n, (D, 1, 1, cfg.H, cfg.W), cfg.dtype)
            out[n] = synth.as_f64(v, cfg.dtype)
        return out

    W = w_planes()

    def one_channel(c):
        x = synth.as_f64(synth.tensor(seed, "x", (1, 1, cfg.H, cfg.W), cfg.dtype, c * HW), cfg.dtype)
        lam = synth.as_f64(synth.tensor(seed, "lam", (D, 1, 1, cfg.H, cfg.W), cfg.dtype, c * HW, HW, cfg.C * HW),
                           cfg.dtype)
        dh = synth.as_f64(synth.tensor(seed, "dh", (D, 1, 1, cfg.H, cfg.W), cfg.dtype, c * HW, HW, cfg.C * HW),
                          cfg.dtype)
        hr = oracle.fwd(x, W["w_l"], W["w_m"], W["w_r"], lam, cfg.dirs, 1)
        gr = oracle.bwd(x, W["w_l"], W["w_m"], W["w_r"], lam, hr, dh, cfg.dirs, 1)
        return c, hr, gr

    sampled = {0, 17, cfg.C - 1}
    dw_sum = [np.zeros((D, 1, 1, cfg.H, cfg.W)) for _ in range(3)]
    tol = TOL[cfg.dtype]
    with ThreadPoolExecutor(max_workers=min(NTHREADS, 16)) as ex:
        for c, hr, gr in ex.map(one_channel, range(cfg.C)):
            for i in range(3):
                dw_sum[i] += gr[1 + i]
            if c in sampled:
                check(test, f"h[c={c}]", from_torch(h[:, 0:1, c:c + 1]), hr, tol)
                check(test, f"dx[c={c}]", from_torch(grads[0][0:1, c:c + 1]), gr[0], tol)
                check(test, f"dlam[c={c}]", from_torch(grads[4][:, 0:1, c:c + 1]), gr[4], tol)
    for i, n in enumerate(("dw_l", "dw_m", "dw_r")):
        check(test, n, from_torch(grads[1 + i]), dw_sum[i], tol)
