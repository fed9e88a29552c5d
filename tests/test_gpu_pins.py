"""GPU pins that need no oracle run, at BASELINE.json's full sizes (SURVEY.md §8(c) "Closed forms",
"Invariants"), plus tiling invariance of the P-split (cluster) path.

* cumsum closed form (w_l = w_r = 0, Eq. 1 with a diagonal step matrix): h is the
  cumulative sum of lam x along the scan; the adjoint g is the reverse cumulative sum of dh, so
  dlam = g x, dx = sum_d g_d lam_d, dw_m = 0 exactly and dw_l = [r>=1] g (h_{t-1}[r-1] - h_{t-1}[r]) / w_m,
  dw_r = [r<=P-2] g (h_{t-1}[r+1] - h_{t-1}[r]) / w_m (the normalisation Jacobian of DESIGN.md §1 with
  l = r = 0). References are torch.cumsum in fp64 of the GPU's own inputs.
* constant input (lam = 1, x = k, row-stochastic taps): h_t = (t + 1) k at every position,
  edges included (R2); an impulse at t = 0 stays constant (h_t = k).
* adjoint mass: with x = lam = 1 and dh = 1 on the last step only, sum_r g_t[r] = P for every t (the
  transpose of a row-stochastic step matrix preserves the sum), and dlam = g.
* GSPN_FLAG_FORCE_SPLIT: the cluster (P-split) path equals the single-CTA path bitwise (fwd h, bwd
  dlam / dx; dw within tolerance where the two use different kernels).
"""
from __future__ import annotations

import os

import pytest

import paper_2512_07884_b200 as gspn
from synth.configs import get_config
from synth.device import make_inputs
from tests.parity_utils import TOL, check, from_torch, host_inputs, record, small_config, to_torch

pytestmark = pytest.mark.gpu


def _to_scan(a, dbit):
    """View the last two dims [H, W] in scan coordinates [t, r] of direction dbit."""
    import torch

    if dbit == gspn.DIR_T2B:
        return a
    if dbit == gspn.DIR_B2T:
        return torch.flip(a, dims=[-2])
    if dbit == gspn.DIR_L2R:
        return a.transpose(-1, -2)
    return torch.flip(a.transpose(-1, -2), dims=[-2])


def _from_scan(a, dbit):
    """Inverse of _to_scan (a new tensor: torch.flip copies)."""
    import torch

    if dbit == gspn.DIR_T2B:
        return a
    if dbit == gspn.DIR_B2T:
        return torch.flip(a, dims=[-2])
    if dbit == gspn.DIR_L2R:
        return a.transpose(-1, -2)
    return torch.flip(a, dims=[-2]).transpose(-1, -2)


def _dirbits(dirs):
    return [b for b in (1, 2, 4, 8) if dirs & b]


def _test_id():
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_cumsum_closed_form_config4(dtype, cuda_device):
    import torch

    cfg = get_config("4").with_(dtype=dtype)
    t = make_inputs(cfg, cuda_device)
    t["w_l"].zero_()
    t["w_r"].zero_()
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], cfg.dirs, cfg.G)
    dx, dwl, dwm, dwr, dlam = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], cfg.dirs, cfg.G)
    torch.cuda.synchronize()
    tol = TOL[dtype]
    test = _test_id()
    assert int(torch.count_nonzero(dwm)) == 0, "dw_m must be exactly 0 when w_l = w_r = 0"
    f64 = torch.float64
    dx_ref = torch.zeros(t["x"].shape, dtype=f64, device=cuda_device)
    err = {"h": 0.0, "dlam": 0.0, "dw_l": 0.0, "dw_r": 0.0}
    for k, dbit in enumerate(_dirbits(cfg.dirs)):
        for b in range(cfg.B):
            x = _to_scan(t["x"][b].to(f64), dbit)
            lam = _to_scan(t["lam"][k, b].to(f64), dbit)
            wm = _to_scan(t["w_m"][k, b].to(f64), dbit)
            dh = _to_scan(t["dh"][k, b].to(f64), dbit)
            href = torch.cumsum(lam * x, dim=-2)
            g = torch.flip(torch.cumsum(torch.flip(dh, dims=[-2]), dim=-2), dims=[-2])
            hp = torch.zeros_like(href)
            hp[:, 1:] = href[:, :-1]                       # h_{t-1}, zero at t = 0
            dwl_ref = torch.zeros_like(href)
            dwr_ref = torch.zeros_like(href)
            dwl_ref[:, :, 1:] = g[:, :, 1:] * (hp[:, :, :-1] - hp[:, :, 1:]) / wm[:, :, 1:]
            dwr_ref[:, :, :-1] = g[:, :, :-1] * (hp[:, :, 1:] - hp[:, :, :-1]) / wm[:, :, :-1]
            got = {"h": _to_scan(h[k, b], dbit), "dlam": _to_scan(dlam[k, b], dbit),
                   "dw_l": _to_scan(dwl[k, b], dbit), "dw_r": _to_scan(dwr[k, b], dbit)}
            ref = {"h": href, "dlam": g * x, "dw_l": dwl_ref, "dw_r": dwr_ref}
            for n in err:
                e = float((got[n].to(f64) - ref[n]).abs().max() / ref[n].abs().max())
                err[n] = max(err[n], e)
                assert e <= tol, f"{n} dir {dbit:#x} b {b}: normwise {e:.3e} > {tol}"
            dx_ref[b] += _from_scan(g * lam, dbit)
    e = float((dx.to(f64) - dx_ref).abs().max() / dx_ref.abs().max())
    err["dx"] = e
    for n, v in err.items():
        record(test, n, v, tol)  # max over direction slabs and batches
    assert e <= tol, f"dx normwise {e:.3e}"


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_constant_and_impulse_inputs_config4(dtype, cuda_device):
    import torch

    cfg = get_config("4").with_(dtype=dtype)
    t = make_inputs(cfg, cuda_device, with_dh=False)
    lam = torch.ones_like(t["lam"])
    x = torch.full_like(t["x"], 0.5)
    h = gspn.fwd(x, t["w_l"], t["w_m"], t["w_r"], lam, cfg.dirs, cfg.G)
    tol = TOL[dtype]
    test = _test_id()
    f64 = torch.float64
    for k, dbit in enumerate(_dirbits(cfg.dirs)):
        hs = _to_scan(h[k], dbit).to(f64)                    # [B, C, L, P]
        L = hs.shape[-2]
        ref = 0.5 * torch.arange(1, L + 1, dtype=f64, device=cuda_device).view(L, 1)
        e = float((hs - ref).abs().max() / ref.abs().max())
        record(test, f"h_const[{dbit:#x}]", e, tol)
        assert e <= tol, f"constant input, dir {dbit:#x}: {e:.3e}"
    # impulse at the first scan step of every direction: x = 0.5 on that row / column only
    for k, dbit in enumerate(_dirbits(cfg.dirs)):
        xs = torch.zeros_like(_to_scan(t["x"], dbit))
        xs[..., 0, :] = 0.5
        xi = _from_scan(xs, dbit).contiguous()
        sl = slice(k, k + 1)
        hi = gspn.fwd(xi, t["w_l"][sl].contiguous(), t["w_m"][sl].contiguous(), t["w_r"][sl].contiguous(),
                      lam[sl].contiguous(), dbit, cfg.G)
        e = float((_to_scan(hi[0], dbit).to(f64) - 0.5).abs().max() / 0.5)
        record(test, f"h_impulse[{dbit:#x}]", e, tol)
        assert e <= tol, f"impulse, dir {dbit:#x}: {e:.3e}"


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_adjoint_mass_config4(dtype, cuda_device):
    import torch

    cfg = get_config("4").with_(dtype=dtype)
    t = make_inputs(cfg, cuda_device, with_dh=False)
    one_l = torch.ones_like(t["lam"])
    x = torch.ones_like(t["x"])
    dh = torch.zeros_like(t["lam"])
    for k, dbit in enumerate(_dirbits(cfg.dirs)):
        ds = torch.zeros_like(_to_scan(dh[k], dbit))
        ds[..., -1, :] = 1.0
        dh[k] = _from_scan(ds, dbit)
    h = gspn.fwd(x, t["w_l"], t["w_m"], t["w_r"], one_l, cfg.dirs, cfg.G)
    _, _, _, _, dlam = gspn.bwd(x, t["w_l"], t["w_m"], t["w_r"], one_l, h, dh, cfg.dirs, cfg.G)
    tol = TOL[dtype]
    test = _test_id()
    for k, dbit in enumerate(_dirbits(cfg.dirs)):
        g = _to_scan(dlam[k], dbit).to(torch.float64)           # [B, C, L, P]
        P = g.shape[-1]
        e = float((g.sum(dim=-1) - P).abs().max() / P)
        record(test, f"mass[{dbit:#x}]", e, tol)
        assert e <= tol, f"adjoint mass, dir {dbit:#x}: {e:.3e}"


# (B, C, G, H, W, dirs, dtype): per-channel (packed and unpacked), grouped, fp32, ragged P
SPLIT_SHAPES = [
    (1, 3, 3, 200, 136, 0xF, "bf16"),
    (2, 4, 2, 96, 160, 0xF, "bf16"),
    (1, 2, 2, 300, 264, 0xF, "bf16"),
    (1, 2, 1, 100, 120, 0xF, "f32"),
    (1, 2, 2, 512, 512, 0xF, "bf16"),
]


@pytest.mark.parametrize("shape", SPLIT_SHAPES, ids=lambda s: "B{}C{}G{}H{}W{}d{:x}{}".format(*s))
def test_cluster_split_bitwise(shape, cuda_device):
    import torch

    B, C, G, H, W, dirs, dt = shape
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=610)
    t = {n: to_torch(v[0], dt, cuda_device) for n, v in host_inputs(cfg).items()}
    args = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])
    h1 = gspn.fwd(*args, dirs, G)
    p1 = gspn.last_path()
    h2 = gspn.fwd(*args, dirs, G, flags=gspn.FLAG_FORCE_SPLIT)
    assert gspn.last_path() == "stream-cluster" and p1 == "stream", (p1, gspn.last_path())
    assert torch.equal(h1, h2), "cluster-split forward differs from the single-CTA forward"
    g1 = gspn.bwd(*args, h1, t["dh"], dirs, G)
    g2 = gspn.bwd(*args, h1, t["dh"], dirs, G, flags=gspn.FLAG_FORCE_SPLIT)
    assert gspn.last_path() == "stream-cluster"
    assert torch.equal(g1[4], g2[4]), "dlam differs"
    assert torch.equal(g1[0], g2[0]), "dx differs"
    for i, n in ((1, "dw_l"), (2, "dw_m"), (3, "dw_r")):
        if G < C:  # both use the split backward: same kernels downstream of g
            assert torch.equal(g1[i], g2[i]), f"{n} differs"
        else:      # fused (vertical dw in the recurrence) vs output-kernel Jacobian: same math, other grouping
            check(_test_id(), n, from_torch(g2[i]), from_torch(g1[i]), TOL[dt])
