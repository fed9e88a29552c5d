"""GPU parity of the SURVEY §8(f) rows against the fp64 oracle (through the C ABI):

NEXT-1  gspn_merge_fwd / gspn_merge_bwd (output gate + direction merge, Eq. 2);
        standalone, composed with the scan (fwd -> merge, merge adjoint -> bwd), and at BASELINE config 4's
        full size on sampled outputs.

Inputs come from synth on the host (never from the CUDA path); tolerances are north_star's normwise
1e-5 (fp32) / 2e-2 (bf16) (R16), with the stored-dtype intermediates of DESIGN.md R18.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2512_07884_b200 as gspn
import synth
from tests.parity_utils import TOL, check, from_torch, host_inputs, host_tensor, normwise, round_io, small_config, to_torch

pytestmark = pytest.mark.gpu


def _dev():
    import torch

    return torch.device("cuda:0")


# (B, C, H, W, dirs, dtype): N % 8 == 0 (vector kernels) and N % 8 != 0 (scalar kernels), D = 1..4
MERGE_SHAPES = [
    (2, 4, 16, 16, 0xF, "bf16"),
    (2, 4, 16, 16, 0xF, "f32"),
    (1, 3, 5, 7, 0xF, "bf16"),
    (1, 3, 5, 7, 0x5, "f32"),
    (3, 2, 9, 11, 0x1, "bf16"),
    (1, 8, 56, 56, 0x7, "bf16"),
    (1, 1, 1, 1, 0xF, "f32"),
]


@pytest.mark.parametrize("mean", [False, True])
@pytest.mark.parametrize("shape", MERGE_SHAPES, ids=lambda s: "B{}C{}H{}W{}d{:x}{}".format(*s))
def test_merge_parity(shape, mean):
    B, C, H, W, dirs, dt = shape
    cfg = small_config(B, C, C, H, W, dirs, dt, cfg_id=601)
    D = cfg.D
    seed = synth.seed_for(cfg.cfg_id)
    hv, hf = host_tensor(cfg, "hs", (D, B, C, H, W))
    uv, uf = host_tensor(cfg, "u", (D, B, C, H, W))
    gv, gf = host_tensor(cfg, "dy", (B, C, H, W))
    assert seed == synth.seed_for(601)
    dev = _dev()
    h, u, dy = to_torch(hv, dt, dev), to_torch(uv, dt, dev), to_torch(gv, dt, dev)
    y = gspn.merge_fwd(h, u, dirs, mean)
    assert gspn.last_path() == "merge" and gspn.last_launch_count() == 1
    dh, du = gspn.merge_bwd(h, u, dy, dirs, mean)
    y_ref = oracle.merge_fwd(hf, uf, mean)
    dh_ref, du_ref = oracle.merge_bwd(hf, uf, gf, mean)
    tol = TOL[dt]
    assert normwise(from_torch(y), y_ref) <= tol
    for k in range(D):
        assert normwise(from_torch(dh)[k], dh_ref[k]) <= tol
        assert normwise(from_torch(du)[k], du_ref[k]) <= tol


@pytest.mark.parametrize("shape", [(2, 4, 2, 40, 56, 0xF, "bf16"), (1, 3, 3, 17, 33, 0xF, "f32"),
                                   (1, 4, 1, 64, 64, 0xF, "bf16")], ids=str)
def test_scan_then_merge_end_to_end(shape):
    """y = merge(fwd(...)); the adjoint chain dy -> (dh, du) -> gspn_bwd -> (dx, dw, dlam), against the
    oracle chain evaluated on the stored-dtype intermediates (h and dh as the API stores them, R18)."""
    B, C, G, H, W, dirs, dt = shape
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=602)
    inp = host_inputs(cfg)
    f = {k: v[1] for k, v in inp.items()}
    uv, uf = host_tensor(cfg, "u", (cfg.D, B, C, H, W))
    gv, gf = host_tensor(cfg, "dy", (B, C, H, W))
    dev = _dev()
    t = {k: to_torch(v[0], dt, dev) for k, v in inp.items()}
    u, dy = to_torch(uv, dt, dev), to_torch(gv, dt, dev)
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G)
    y = gspn.merge_fwd(h, u, dirs)
    dh, du = gspn.merge_bwd(h, u, dy, dirs)
    grads = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, dh, dirs, G)

    h_ref = round_io(oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G), dt)
    y_ref = oracle.merge_fwd(h_ref, uf)
    dh_ref, du_ref = oracle.merge_bwd(h_ref, uf, gf)
    g_ref = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], h_ref, round_io(dh_ref, dt), dirs, G)
    tol = TOL[dt]
    assert normwise(from_torch(y), y_ref) <= tol
    assert normwise(from_torch(du), du_ref) <= tol
    for name, a, r in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), grads, g_ref):
        assert normwise(from_torch(a), r) <= tol, name


def test_merge_fullsize_config4_sampled():
    """BASELINE configs[3] shape (B=4, C=320, 512 x 512, 4 directions, bf16) on device-generated inputs;
    4096 sampled outputs of y, dh and du recomputed by the oracle from host-regenerated values."""
    import torch

    cfg = synth.get_config("4")
    D, B, C, H, W = cfg.D, cfg.B, cfg.C, cfg.H, cfg.W
    N = B * C * H * W
    seed = synth.seed_for(cfg.cfg_id)
    from synth.device import fill_

    dev = _dev()
    h = fill_(torch.empty((D, B, C, H, W), dtype=torch.bfloat16, device=dev), seed, "hs")
    u = fill_(torch.empty((D, B, C, H, W), dtype=torch.bfloat16, device=dev), seed, "u")
    dy = fill_(torch.empty((B, C, H, W), dtype=torch.bfloat16, device=dev), seed, "dy")
    y = gspn.merge_fwd(h, u, 0xF)
    dh, du = gspn.merge_bwd(h, u, dy, 0xF)
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    n = np.concatenate([rng.integers(0, N, 4090), [0, 1, N - 3, N - 2, N - 1, N // 2]]).astype(np.uint64)
    idx = torch.from_numpy(n.astype(np.int64)).to(dev)
    hs = np.stack([synth.as_f64(synth.values(seed, "hs", n + np.uint64(k * N), "bf16"), "bf16") for k in range(D)])
    us = np.stack([synth.as_f64(synth.values(seed, "u", n + np.uint64(k * N), "bf16"), "bf16") for k in range(D)])
    gs = synth.as_f64(synth.values(seed, "dy", n, "bf16"), "bf16")
    y_ref = oracle.merge_fwd(hs, us)
    dh_ref, du_ref = oracle.merge_bwd(hs, us, gs)
    got_y = from_torch(y.reshape(-1)[idx])
    got_dh = from_torch(dh.reshape(D, -1)[:, idx])
    got_du = from_torch(du.reshape(D, -1)[:, idx])
    assert normwise(got_y, y_ref) <= TOL["bf16"]
    assert normwise(got_dh, dh_ref) <= TOL["bf16"]
    assert normwise(got_du, du_ref) <= TOL["bf16"]


# ------------------------------------------------------------------------------------ NEXT-2 kchunk

# (B, C, G, H, W, dirs, dtype, kchunk): stream path (vertical/horizontal, reversed, partial first/last
# tiles, packed small planes, grouped weights, P-split clusters) and segments shorter than, equal to and
# longer than a 16-step tile, with a short last segment; kchunk = 1 (every step isolated).
LOCAL_CASES = [
    (1, 4, 4, 64, 64, 0xF, "bf16", 16),
    (1, 4, 4, 64, 64, 0xF, "bf16", 5),
    (2, 3, 3, 100, 72, 0xF, "bf16", 24),
    (1, 4, 2, 37, 24, 0xF, "bf16", 7),
    (2, 2, 2, 19, 12, 0xF, "f32", 3),
    (1, 2, 2, 40, 56, 0xF, "f32", 8),
    (2, 4, 4, 56, 56, 0xF, "bf16", 14),
    (1, 4, 1, 64, 64, 0xF, "bf16", 32),
    (1, 2, 2, 24, 1000, 0xF, "bf16", 100),
    (1, 1, 1, 700, 48, 0xF, "bf16", 50),
    (1, 2, 2, 33, 17, 0xF, "f32", 4),
    (1, 2, 2, 48, 40, 0xF, "bf16", 1),
    (1, 3, 3, 512, 512, 0xF, "bf16", 64),
]


@pytest.mark.parametrize("flags", [0, gspn.FLAG_FORCE_GENERIC], ids=["auto", "generic"])
@pytest.mark.parametrize("case", LOCAL_CASES, ids=lambda c: "B{}C{}G{}H{}W{}d{:x}{}k{}".format(*c))
def test_local_parity(case, flags):
    B, C, G, H, W, dirs, dt, k = case
    if flags and H * W > 64 * 64 and max(H, W) > 512:
        pytest.skip("generic path on P-split shapes is covered by test_gpu_parity")
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=603)
    inp = host_inputs(cfg)
    f = {n: v[1] for n, v in inp.items()}
    dev = _dev()
    t = {n: to_torch(v[0], dt, dev) for n, v in inp.items()}
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G, flags=flags, kchunk=k)
    path = gspn.last_path()
    grads = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], dirs, G, flags=flags, kchunk=k)
    h_ref = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G, kchunk=k)
    g_ref = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], round_io(h_ref, dt), f["dh"], dirs, G,
                       kchunk=k)
    tol = TOL[dt]
    hg = from_torch(h)
    for s in range(cfg.D):
        assert normwise(hg[s], h_ref[s]) <= tol, f"h slab {s} ({path})"
    for name, a, r in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), grads, g_ref):
        a = from_torch(a)
        if a.ndim == 5:
            for s in range(a.shape[0]):
                assert normwise(a[s], r[s]) <= tol, f"{name} slab {s} ({path})"
        else:
            assert normwise(a, r) <= tol, f"{name} ({path})"
    if not flags and (W * (2 if dt == "bf16" else 4)) % 16 == 0:
        assert path.startswith("stream")


def test_local_kchunk_one_is_lambda_x():
    """kchunk = 1 isolates every step: h = lam x exactly up to the I/O rounding of one product."""
    import torch

    cfg = small_config(2, 4, 4, 64, 64, 0xF, "f32", cfg_id=604)
    inp = host_inputs(cfg)
    dev = _dev()
    t = {n: to_torch(v[0], "f32", dev) for n, v in inp.items()}
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], 0xF, 4, kchunk=1)
    torch.testing.assert_close(h, t["lam"] * t["x"].unsqueeze(0), rtol=0, atol=0)


# ------------------------------------------------------------------- fused backward (G = C, stream path)

# Unpacked, unsplit per-channel shapes (max(H, W) > 256 or a single plane): the adjoint recurrence and
# the tap gradients run in one pass; ragged tiles on both axes, reversed directions, single directions.
FUSED_SHAPES = [
    (1, 2, 2, 300, 264, 0xF, "bf16"),
    (2, 2, 2, 264, 300, 0xF, "f32"),
    (1, 3, 3, 272, 288, 0x5, "bf16"),
    (1, 2, 2, 280, 264, 0xA, "bf16"),
    (1, 1, 1, 100, 72, 0xF, "bf16"),
    (1, 1, 1, 37, 24, 0xF, "f32"),
    (1, 2, 2, 512, 512, 0xF, "bf16"),
    (1, 2, 2, 257, 512, 0xC, "bf16"),
    (1, 2, 2, 512, 8, 0xF, "bf16"),
    (1, 2, 2, 300, 264, 0x3, "bf16"),   # vertical directions only (the output kernel forms dlam, dx only)
    (1, 2, 2, 264, 272, 0x1, "f32"),
    (2, 4, 4, 56, 56, 0xF, "bf16"),     # packed small planes
    (1, 6, 6, 40, 48, 0x6, "f32"),
]


@pytest.mark.parametrize("pre", [False, True], ids=["raw", "prenorm"])
@pytest.mark.parametrize("shape", FUSED_SHAPES, ids=lambda s: "B{}C{}G{}H{}W{}d{:x}{}".format(*s))
def test_fused_bwd_parity(shape, pre):
    """gspn_bwd on the fused path vs the oracle backward given the same (stored-dtype) h."""
    B, C, G, H, W, dirs, dt = shape
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=605)
    inp = host_inputs(cfg)
    f = {n: v[1] for n, v in inp.items()}
    dev = _dev()
    t = {n: to_torch(v[0], dt, dev) for n, v in inp.items()}
    flags = gspn.FLAG_PRENORMALIZED if pre else 0
    if pre:  # pre-normalised taps: use the oracle's normalisation of the generated taps as the input
        import torch

        S = t["w_l"].float() + t["w_m"].float() + t["w_r"].float()
        for n in ("w_l", "w_m", "w_r"):
            t[n] = (t[n].float() / S).to(t[n].dtype)
            f[n] = from_torch(t[n])
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G, flags=flags)
    grads = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], dirs, G, flags=flags)
    assert gspn.last_path() == "stream-fused"
    oflags = oracle.PRENORMALIZED if pre else 0
    h_ref = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G, flags=oflags)
    g_ref = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], from_torch(h), f["dh"], dirs, G,
                       flags=oflags)
    tol = TOL[dt]
    check("fused_bwd", "h", from_torch(h), h_ref, tol)
    for name, a, r in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), grads, g_ref):
        a = from_torch(a)
        if a.ndim == 5:
            for s in range(a.shape[0]):
                assert normwise(a[s], r[s]) <= tol, f"{name} slab {s}"
        else:
            assert normwise(a, r) <= tol, name


# ------------------------------------------------------------------- small-plane path (max(H, W) <= 32)

# Rows too short for TMA (W s % 16 != 0): BASELINE configs[2]'s 28 x 28 proxy planes, grouped and per
# channel, odd sizes, single directions, GSPN-local.
SMALL_CASES = [
    (2, 8, 1, 28, 28, 0xF, "bf16", 0),
    (2, 12, 4, 28, 28, 0xF, "bf16", 0),
    (1, 6, 6, 28, 26, 0xF, "f32", 0),
    (3, 4, 2, 13, 27, 0xF, "bf16", 0),
    (1, 3, 3, 31, 5, 0x9, "f32", 0),
    (1, 2, 1, 1, 19, 0xF, "bf16", 0),
    (2, 8, 1, 28, 28, 0xF, "bf16", 7),
    (1, 4, 4, 21, 30, 0xF, "f32", 4),
]


@pytest.mark.parametrize("case", SMALL_CASES, ids=lambda c: "B{}C{}G{}H{}W{}d{:x}{}k{}".format(*c))
def test_small_plane_parity(case):
    B, C, G, H, W, dirs, dt, k = case
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=606)
    inp = host_inputs(cfg)
    f = {n: v[1] for n, v in inp.items()}
    dev = _dev()
    t = {n: to_torch(v[0], dt, dev) for n, v in inp.items()}
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G, kchunk=k)
    assert gspn.last_path() == "small"
    grads = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], dirs, G, kchunk=k)
    assert gspn.last_path() == "small"
    h_ref = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G, kchunk=k)
    g_ref = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], from_torch(h), f["dh"], dirs, G, kchunk=k)
    tol = TOL[dt]
    hg = from_torch(h)
    for s in range(cfg.D):
        assert normwise(hg[s], h_ref[s]) <= tol, f"h slab {s}"
    for name, a, r in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), grads, g_ref):
        a = from_torch(a)
        if a.ndim == 5:
            for s in range(a.shape[0]):
                assert normwise(a[s], r[s]) <= tol, f"{name} slab {s}"
        else:
            assert normwise(a, r) <= tol, name


# ------------------------------------------------------------------- NEXT-4 proxy projections

# (B, C, C_proxy, H, W, dtype): BASELINE configs[2] (384 -> 8, 28 x 28) and a configs[4]-like 320 -> 40
PROXY_CASES = [
    (64, 384, 8, 28, 28, "bf16"),
    (2, 320, 40, 16, 24, "bf16"),
    (3, 24, 5, 7, 6, "f32"),
    (1, 8, 8, 4, 4, "f32"),
]


@pytest.mark.parametrize("case", PROXY_CASES, ids=lambda c: "B{}C{}Cp{}H{}W{}{}".format(*c))
def test_proxy_parity(case):
    """down (P [Cp, C]), up (Q [C, Cp]), the data gradients (transposed mixes) and both weight gradients
    against the fp64 oracle on host-generated inputs and weights."""
    import torch

    B, C, Cp, H, W, dt = case
    rng = np.random.default_rng(C + Cp)
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    dev = _dev()

    def mk(shape, scale=1.0):
        a = torch.from_numpy(rng.uniform(-scale, scale, shape)).to(dtype)
        return a.to(dev), a.double().numpy()

    x, xf = mk((B, C, H, W))
    P, Pf = mk((Cp, C), 1.0 / np.sqrt(C))
    Q, Qf = mk((C, Cp), 1.0 / np.sqrt(Cp))
    dy, dyf = mk((B, C, H, W))
    xp = gspn.proxy_mix(x, P)
    assert gspn.last_path().startswith("proxy")
    y = gspn.proxy_mix(xp, Q)
    dxp = gspn.proxy_mix(dy, Q, transpose=True)           # d(up)/d(input) = Q^T dy
    dx = gspn.proxy_mix(dxp, P, transpose=True)           # d(down)/d(input) = P^T dxp
    dQ = gspn.proxy_wgrad(dy, xp)
    dP = gspn.proxy_wgrad(dxp, x)
    torch.cuda.synchronize()
    tol = TOL[dt]
    xp_ref = oracle.proxy_mix(xf, Pf)
    xp_st = from_torch(xp)                                # downstream refs on the stored-dtype values (R18)
    assert normwise(xp_st, xp_ref) <= tol
    assert normwise(from_torch(y), oracle.proxy_mix(xp_st, Qf)) <= tol
    dxp_st = from_torch(dxp)
    assert normwise(dxp_st, oracle.proxy_mix(dyf, Qf.T)) <= tol
    assert normwise(from_torch(dx), oracle.proxy_mix(dxp_st, Pf.T)) <= tol
    assert normwise(from_torch(dQ), oracle.proxy_wgrad(dyf, xp_st)) <= tol
    assert normwise(from_torch(dP), oracle.proxy_wgrad(dxp_st, xf)) <= tol


@pytest.mark.parametrize("shape", [(1, 2, 2, 300, 264, 0xF, "bf16", 50), (2, 4, 4, 56, 56, 0xF, "f32", 20)],
                         ids=lambda s: "B{}C{}G{}H{}W{}d{:x}{}k{}".format(*s))
def test_fused_local_prenormalized(shape):
    """Hybrid fused backward with GSPN-local segments and pre-normalised taps together."""
    import torch

    B, C, G, H, W, dirs, dt, k = shape
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=607)
    inp = host_inputs(cfg)
    f = {n: v[1] for n, v in inp.items()}
    dev = _dev()
    t = {n: to_torch(v[0], dt, dev) for n, v in inp.items()}
    S = t["w_l"].float() + t["w_m"].float() + t["w_r"].float()
    for n in ("w_l", "w_m", "w_r"):
        t[n] = (t[n].float() / S).to(t[n].dtype)
        f[n] = from_torch(t[n])
    fl = gspn.FLAG_PRENORMALIZED
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G, flags=fl, kchunk=k)
    grads = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], dirs, G, flags=fl, kchunk=k)
    assert gspn.last_path() == "stream-fused"
    h_ref = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G, flags=oracle.PRENORMALIZED,
                       kchunk=k)
    g_ref = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], from_torch(h), f["dh"], dirs, G,
                       flags=oracle.PRENORMALIZED, kchunk=k)
    tol = TOL[dt]
    assert normwise(from_torch(h), h_ref) <= tol
    for name, a, r in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), grads, g_ref):
        assert normwise(from_torch(a), r) <= tol, name
    torch.cuda.synchronize()


# (B, Ci, Co, H, W): the configs' compact blocks (320 -> 40 -> 320, 384 -> 8 -> 384) and ragged ones: K not a
# multiple of 64, Co not a multiple of 128 (1, 2 and 4 M tiles), a partial last pixel tile
UMMA_CASES = [
    (2, 320, 40, 16, 24),
    (2, 40, 320, 16, 24),
    (3, 384, 8, 28, 28),
    (3, 8, 384, 28, 28),
    (1, 100, 7, 8, 17 * 8),
    (3, 64, 130, 8, 8),
    (1, 24, 500, 4, 16),
    (2, 200, 256, 12, 12),
]


@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("case", UMMA_CASES, ids=lambda c: "B{}Ci{}Co{}H{}W{}".format(*c))
def test_proxy_umma_parity(case, trans):
    """gspn_proxy_mix on tcgen05 (path "proxy-umma") vs the fp64 oracle on the same bf16 inputs, and vs the
    SIMT kernel (GSPN_FLAG_PROXY_SIMT) on the same call."""
    import torch

    B, Ci, Co, H, W = case
    rng = np.random.default_rng(Ci * 1000 + Co)
    dev = _dev()
    x = torch.from_numpy(rng.uniform(-1, 1, (B, Ci, H, W))).to(torch.bfloat16)
    Mw = torch.from_numpy(rng.uniform(-1, 1, (Ci, Co) if trans else (Co, Ci)) / np.sqrt(Ci)).to(torch.bfloat16)
    y = gspn.proxy_mix(x.to(dev), Mw.to(dev), transpose=trans)
    assert gspn.last_path() == "proxy-umma"
    ys = None
    if Ci * Co <= 49152:  # the SIMT kernel stages M in shared memory
        ys = gspn.proxy_mix(x.to(dev), Mw.to(dev), transpose=trans, simt=True)
        assert gspn.last_path() == "proxy"
    Mf = Mw.double().numpy()
    ref = oracle.proxy_mix(x.double().numpy(), Mf.T if trans else Mf)
    check("proxy_umma", "out", from_torch(y), ref, TOL["bf16"], per_slab=False)
    if ys is not None:
        check("proxy_umma", "out vs simt", from_torch(y), from_torch(ys), TOL["bf16"], per_slab=False)
    if not trans:  # weight gradient of this projection: dM = dout in^T over every pixel (tcgen05, K = B H W)
        dout = torch.from_numpy(rng.uniform(-1, 1, (B, Co, H, W))).to(torch.bfloat16)
        dM = gspn.proxy_wgrad(dout.to(dev), x.to(dev))
        assert gspn.last_path() == "proxy-umma"
        check("proxy_umma", "wgrad", from_torch(dM), oracle.proxy_wgrad(dout.double().numpy(), x.double().numpy()),
              TOL["bf16"], per_slab=False)


def test_proxy_umma_config5_block_sampled():
    """BASELINE configs[4]'s compact block at full size: 320 -> 40 (down) and 40 -> 320 (up) over 2048^2
    pixels on tcgen05; 2048 sampled pixels of every output channel recomputed in fp64 on the host."""
    import torch

    B, C, Cp, H, W = 1, 320, 40, 2048, 2048
    dev = _dev()
    g = torch.Generator(device=dev).manual_seed(5)
    x = (torch.rand((B, C, H, W), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    P = ((torch.rand((Cp, C), generator=g, device=dev) * 2 - 1) / C ** 0.5).to(torch.bfloat16)
    Q = ((torch.rand((C, Cp), generator=g, device=dev) * 2 - 1) / Cp ** 0.5).to(torch.bfloat16)
    xp = gspn.proxy_mix(x, P)
    assert gspn.last_path() == "proxy-umma"
    y = gspn.proxy_mix(xp, Q)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    pix = np.concatenate([rng.integers(0, H * W, 2042), [0, 1, 255, 256, H * W - 2, H * W - 1]])
    idx = torch.from_numpy(pix).to(dev)
    xs = x.reshape(C, -1)[:, idx].double().cpu().numpy()            # [C, S]
    xps = xp.reshape(Cp, -1)[:, idx].double().cpu().numpy()         # GPU xp (stored bf16) at those pixels
    Pf, Qf = P.double().cpu().numpy(), Q.double().cpu().numpy()
    check("proxy_umma_cfg5", "down", xps, Pf @ xs, TOL["bf16"], per_slab=False)
    ys = y.reshape(C, -1)[:, idx].double().cpu().numpy()
    check("proxy_umma_cfg5", "up", ys, Qf @ xps, TOL["bf16"], per_slab=False)


# ------------------------------------------------------------------- NEXT-1 merged backward

# (B, C, G, H, W, dirs, dtype, expected path): the fused single launch (per-channel: unpacked, packed, fp32,
# single directions) and the unfused fallback (grouped, small planes)
MERGED_CASES = [
    (1, 2, 2, 300, 264, 0xF, "bf16", "stream-fused-merged"),
    (2, 4, 4, 56, 56, 0xF, "bf16", "stream-fused-merged"),
    (1, 2, 2, 512, 512, 0xF, "bf16", "stream-fused-merged"),
    (2, 2, 2, 264, 300, 0xF, "f32", "stream-fused-merged"),
    (1, 3, 3, 272, 288, 0x5, "bf16", "stream-fused-merged"),
    (1, 2, 2, 300, 264, 0xA, "f32", "stream-fused-merged"),
    (2, 4, 2, 40, 56, 0xF, "bf16", "merged-unfused"),
    (2, 8, 1, 28, 28, 0xF, "bf16", "merged-unfused"),
]


@pytest.mark.parametrize("mean", [False, True], ids=["sum", "mean"])
@pytest.mark.parametrize("case", MERGED_CASES, ids=lambda c: "B{}C{}G{}H{}W{}d{:x}{}".format(*c[:7]))
def test_bwd_merged_parity(case, mean):
    """gspn_bwd_merged (dh = s u dy formed in the backward launch, du written) against the oracle chain
    merge adjoint -> scan adjoint (Eq. 2) on the GPU's own stored h (R18)."""
    B, C, G, H, W, dirs, dt, want = case
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=608)
    inp = host_inputs(cfg)
    f = {n: v[1] for n, v in inp.items()}
    uv, uf = host_tensor(cfg, "u", (cfg.D, B, C, H, W))
    gv, gf = host_tensor(cfg, "dy", (B, C, H, W))
    dev = _dev()
    t = {n: to_torch(v[0], dt, dev) for n, v in inp.items()}
    u, dy = to_torch(uv, dt, dev), to_torch(gv, dt, dev)
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G)
    outs = gspn.bwd_merged(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, u, dy, dirs, G, mean=mean)
    assert gspn.last_path() == want, gspn.last_path()
    if want == "stream-fused-merged":
        assert gspn.last_launch_count() == 1
    hs = from_torch(h)
    dh_ref, du_ref = oracle.merge_bwd(hs, uf, gf, mean)
    g_ref = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], hs, dh_ref, dirs, G)
    tol = TOL[dt]
    for name, a, r in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam", "du"), outs, list(g_ref) + [du_ref]):
        check("bwd_merged", name, from_torch(a), r, tol)


FWD_MERGED_CASES = [
    (1, 2, 2, 300, 264, 0xF, "bf16", "stream-merged"),
    (2, 4, 4, 56, 56, 0xF, "bf16", "stream-merged"),
    (2, 3, 1, 64, 80, 0xF, "f32", "stream-merged"),
    (1, 2, 2, 24, 1000, 0xF, "bf16", "merged-unfused"),   # P-split chains: scan then merge
    (2, 8, 1, 28, 28, 0x9, "bf16", "merged-unfused"),     # small planes
]


@pytest.mark.parametrize("keep_h", [True, False], ids=["h", "noh"])
@pytest.mark.parametrize("mean", [False, True], ids=["sum", "mean"])
@pytest.mark.parametrize("case", FWD_MERGED_CASES, ids=lambda c: "B{}C{}G{}H{}W{}d{:x}{}".format(*c[:7]))
def test_fwd_merged_parity(case, mean, keep_h):
    """gspn_fwd_merged: y = s sum_d u_d h_d from the scan's own h in the same launch, vs the
    oracle merge of the oracle forward; h (when kept) vs the oracle forward."""
    B, C, G, H, W, dirs, dt, want = case
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=609)
    inp = host_inputs(cfg)
    f = {n: v[1] for n, v in inp.items()}
    uv, uf = host_tensor(cfg, "u", (cfg.D, B, C, H, W))
    dev = _dev()
    t = {n: to_torch(v[0], dt, dev) for n, v in inp.items()}
    u = to_torch(uv, dt, dev)
    y, h = gspn.fwd_merged(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], u, dirs, G, mean=mean, keep_h=keep_h)
    assert gspn.last_path() == want, gspn.last_path()
    if want == "stream-merged":
        assert gspn.last_launch_count() == 1
    h_ref = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G)
    tol = TOL[dt]
    check("fwd_merged", "y", from_torch(y), oracle.merge_fwd(h_ref, uf, mean), tol, per_slab=False)
    if keep_h:
        check("fwd_merged", "h", from_torch(h), h_ref, tol)


# ------------------------------------------------------------------- NEXT-3 recompute-h backward

# (B, C, G, H, W, dirs, dtype, fwd path, bwd path): checkpointed shapes (unpacked, unsplit, H and W multiples
# of the 32-byte tile) and the fallbacks (grouped, packed small planes, P-split)
RECOMPUTE_CASES = [
    (1, 2, 2, 512, 512, 0xF, "bf16", "stream-ckpt", "stream-recompute"),
    (1, 2, 2, 320, 288, 0xF, "bf16", "stream-ckpt", "stream-recompute"),
    (2, 2, 2, 264, 272, 0xF, "f32", "stream-ckpt", "stream-recompute"),
    (1, 3, 3, 288, 320, 0x5, "bf16", "stream-ckpt", "stream-recompute"),
    (1, 2, 2, 272, 288, 0xA, "f32", "stream-ckpt", "stream-recompute"),
    (2, 4, 2, 40, 56, 0xF, "bf16", "ckpt-deferred", "recompute-unfused"),
    (2, 4, 4, 56, 56, 0xF, "bf16", "ckpt-deferred", "recompute-unfused"),
    (1, 2, 2, 24, 1000, 0xF, "bf16", "ckpt-deferred", "recompute-unfused"),
]


@pytest.mark.parametrize("case", RECOMPUTE_CASES, ids=lambda c: "B{}C{}G{}H{}W{}d{:x}{}".format(*c[:7]))
def test_recompute_bwd_parity(case):
    """gspn_fwd_ckpt (checkpoints, no h) -> gspn_bwd_recompute vs the oracle backward on the oracle's own
    UNROUNDED h: the recompute sees h in fp32, so even bf16 dw is held to the unrounded reference (cf. R18)."""
    import torch

    B, C, G, H, W, dirs, dt, fpath, bpath = case
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=611)
    inp = host_inputs(cfg)
    f = {n: v[1] for n, v in inp.items()}
    dev = _dev()
    t = {n: to_torch(v[0], dt, dev) for n, v in inp.items()}
    a = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])
    ckpt, _ = gspn.fwd_ckpt(*a, dirs, G)
    assert gspn.last_path() == fpath, gspn.last_path()
    grads = gspn.bwd_recompute(*a, ckpt, t["dh"], dirs, G)
    assert gspn.last_path() == bpath, gspn.last_path()
    if bpath == "stream-recompute":
        assert gspn.last_launch_count() == 1
    h_ref = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G)
    g_ref = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], h_ref, f["dh"], dirs, G)
    tol = TOL[dt]
    for name, got, ref in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), grads, g_ref):
        check("recompute_bwd", name, from_torch(got), ref, tol)
    # the checkpointing forward computes the same h as gspn_fwd (when it is kept)
    ck2, hk = gspn.fwd_ckpt(*a, dirs, G, keep_h=True)
    h0 = gspn.fwd(*a, dirs, G)
    assert torch.equal(hk, h0)


def test_recompute_dw_error_at_l2048():
    """dw at L = 2048 (H = 2048, W = 512, vertical directions: P = 512 fits one CTA) through the saved-h
    backward and through the recompute backward, both against the oracle on its own unrounded h; the
    recompute path sees fp32 h, so its bf16 dw error must not exceed the saved-h path's."""
    B, C, G, H, W, dirs, dt = 1, 2, 2, 2048, 512, 0x3, "bf16"
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=612)
    inp = host_inputs(cfg)
    f = {n: v[1] for n, v in inp.items()}
    dev = _dev()
    t = {n: to_torch(v[0], dt, dev) for n, v in inp.items()}
    a = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])
    h = gspn.fwd(*a, dirs, G)
    g_saved = gspn.bwd(*a, h, t["dh"], dirs, G)
    ckpt, _ = gspn.fwd_ckpt(*a, dirs, G)
    g_rc = gspn.bwd_recompute(*a, ckpt, t["dh"], dirs, G)
    assert gspn.last_path() == "stream-recompute"
    h_ref = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G, threads=oracle.default_threads())
    g_ref = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], h_ref, f["dh"], dirs, G,
                       threads=oracle.default_threads())
    for i, name in ((1, "dw_l"), (2, "dw_m"), (3, "dw_r")):
        e_saved = check("L2048_saved_h", name, from_torch(g_saved[i]), g_ref[i], TOL[dt])
        e_rc = check("L2048_recompute", name, from_torch(g_rc[i]), g_ref[i], TOL[dt])
        assert e_rc <= e_saved * 1.05, (name, e_rc, e_saved)


def test_experiment_hf_backward_matches_default():
    """The kHF backward (GSPN_EXPERIMENTS + GSPN_HF: horizontal dw in the recurrence; measured slower, kept
    as an experiment) agrees with the default hybrid within the dtype tolerance -- packed fp32, unpacked
    bf16 with a ragged P, config-4-like, grouped-free 3-channel shapes. Runs in a child process: the
    experiment knobs are read from the environment once per process."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "hf_cmp.py"), "1,8,8,16,16,15,f32",
                        "1,2,2,300,264,15,bf16", "2,2,2,512,512,15,bf16", "1,3,3,200,136,15,bf16"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]


@pytest.mark.gpu
def test_segment_items_bitwise_equal_global_schedule():
    """NEXT-2 as a scheduler: GSPN-local segments as independent work items give the same
    bits as the same kchunk run chain by chain -- packed small planes, an unpacked bf16 plane with a short last
    segment, grouped weights on the split backward, fp32, and a P-split (cluster) chain. Child process: the
    experiment knob that turns segment items off is read from the environment."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "seg_cmp.py"), "1,8,8,64,64,15,bf16,16",
                        "1,2,2,512,512,15,bf16,128", "1,2,2,400,336,15,bf16,96", "1,4,1,256,256,15,bf16,64",
                        "1,2,2,128,96,15,f32,32", "1,2,1,1040,1040,15,bf16,256"],
                       capture_output=True, text=True, timeout=900, cwd=root)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
