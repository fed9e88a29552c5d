"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Inputs are generated on the host by synth (never read back from the CUDA path) and uploaded; the
tolerance is BASELINE.json's north_star: normwise max|gpu - ref| / max|ref| <= 1e-5 (fp32 I/O) and
<= 2e-2 (bf16 I/O), per output tensor and per direction slab (R16).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2512_07884_b200 as gspn
from tests.parity_utils import (TOL, check, from_torch, record, host_inputs, io_from_f64, normwise, round_io, small_config,
                                to_torch)

pytestmark = pytest.mark.gpu

NTHREADS = oracle.default_threads()

# (B, C, G, H, W, dirs, dtype): ragged tails, degenerate H/W = 1, groups 1 < G < C, single and mixed
# directions, several tiles along L and P, P above one CTA's thread count.
SHAPES = [
    (1, 8, 8, 16, 16, 0x4, "f32"),     # config 1 (BASELINE configs[0])
    (2, 3, 3, 17, 33, 0xF, "f32"),
    (2, 3, 3, 17, 33, 0xF, "bf16"),
    (1, 4, 1, 9, 5, 0xF, "bf16"),
    (2, 6, 2, 12, 7, 0xF, "f32"),
    (1, 2, 2, 1, 37, 0xF, "f32"),
    (1, 2, 2, 23, 1, 0xF, "bf16"),
    (1, 1, 1, 1, 1, 0xF, "f32"),
    (1, 2, 1, 40, 1100, 0x5, "f32"),
    (3, 5, 5, 64, 64, 0xA, "bf16"),
    (1, 4, 4, 56, 56, 0xF, "bf16"),
    (2, 8, 1, 28, 28, 0xF, "bf16"),
    (1, 2, 2, 96, 80, 0xF, "f32"),
    (1, 2, 2, 256, 256, 0xF, "bf16"),
    (1, 3, 3, 512, 512, 0xF, "bf16"),
    (1, 2, 1, 200, 136, 0xF, "bf16"),
    # stream-path ragged cases: partial first/last tiles, P not a multiple of a warp's span,
    # P near the 512-position tile, tiny P against large L
    (2, 3, 3, 100, 72, 0xF, "bf16"),
    (1, 4, 2, 37, 24, 0xF, "bf16"),
    (2, 2, 2, 19, 12, 0xF, "f32"),
    (1, 2, 2, 512, 8, 0xF, "bf16"),
    (1, 2, 1, 8, 512, 0xF, "f32"),
    (1, 2, 2, 500, 504, 0xF, "bf16"),
    (1, 1, 1, 250, 248, 0xF, "bf16"),
    # P-split over a thread-block cluster (P > 512: 2-3 CTAs per chain, ghosts through DSMEM)
    (1, 2, 2, 24, 1000, 0xF, "bf16"),
    (1, 1, 1, 700, 48, 0xF, "bf16"),
    (1, 2, 2, 20, 1040, 0xF, "f32"),
    # output phase with whole image rows per TMA box (W > 256, W % 256 == 0: 3 and 5 boxes of 256 per row),
    # per-channel (single-launch backward) and grouped (grouped output kernel, P-split recurrence)
    (1, 2, 2, 24, 768, 0xF, "bf16"),
    (1, 4, 1, 20, 1280, 0xF, "bf16"),
]
FLAGS = [0, gspn.FLAG_FORCE_GENERIC]


def _ids(s):
    return "B{}C{}G{}H{}W{}d{:x}{}".format(*s)


def _upload(inp, dtype, device):
    return {k: to_torch(v[0], dtype, device) for k, v in inp.items()}


def _check(name, got, ref, dtype, per_slab=True):
    import os

    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    check(test, name, got, ref, TOL[dtype], per_slab)


@pytest.fixture(scope="module")
def oracle_cache():
    return {}


def _oracle(shape, cache):
    if shape in cache:
        return cache[shape]
    B, C, G, H, W, dirs, dtype = shape
    cfg = small_config(B, C, G, H, W, dirs, dtype, cfg_id=100 + len(cache))
    inp = host_inputs(cfg)
    f = {k: v[1] for k, v in inp.items()}
    h = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], dirs, G, threads=NTHREADS)
    h_in = round_io(h, dtype)  # oracle h rounded to the I/O dtype: the bwd-given-h input
    g_given = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], h_in, f["dh"], dirs, G, threads=NTHREADS)
    g_e2e = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], h, f["dh"], dirs, G, threads=NTHREADS)
    cache[shape] = (cfg, inp, h, h_in, g_given, g_e2e)
    return cache[shape]


@pytest.mark.parametrize("flags", FLAGS, ids=["default", "generic"])
@pytest.mark.parametrize("shape", SHAPES, ids=_ids)
def test_fwd_parity(shape, flags, cuda_device, oracle_cache):
    B, C, G, H, W, dirs, dtype = shape
    cfg, inp, h_ref, _, _, _ = _oracle(shape, oracle_cache)
    t = _upload(inp, dtype, cuda_device)
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G, flags=flags)
    _check("h", from_torch(h), h_ref, dtype)


@pytest.mark.parametrize("flags", FLAGS, ids=["default", "generic"])
@pytest.mark.parametrize("shape", SHAPES, ids=_ids)
def test_bwd_parity_given_h(shape, flags, cuda_device, oracle_cache):
    B, C, G, H, W, dirs, dtype = shape
    cfg, inp, _, h_in, g_ref, _ = _oracle(shape, oracle_cache)
    t = _upload(inp, dtype, cuda_device)
    h = to_torch(io_from_f64(h_in, dtype), dtype, cuda_device)
    outs = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], dirs, G, flags=flags)
    for name, got, ref in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), outs, g_ref):
        _check(name, from_torch(got), ref, dtype)


@pytest.mark.parametrize("shape", SHAPES, ids=_ids)
def test_fwd_bwd_end_to_end(shape, cuda_device, oracle_cache):
    """GPU fwd -> GPU bwd (on the GPU's own stored h) against the oracle backward on the oracle's own,
    UNROUNDED fp64 h: the I/O-dtype storage of h is charged to the GPU path.
    Exception (R18, measured): bf16 dw is a difference of neighbouring h values scaled by the
    normalisation Jacobian, so the bf16 rounding of the stored h alone moves it by up to 2.2e-2 normwise
    on narrow planes (P = 8, L = 512: neighbours nearly equal after many row-stochastic steps); bf16 dw is
    held to the tolerance against the backward on the stored-dtype h and its unrounded error is logged.
    The bwd-given-h test above isolates the backward kernel on identical h."""
    import os

    B, C, G, H, W, dirs, dtype = shape
    cfg, inp, h_ref, _, g_stored, g_ref = _oracle(shape, oracle_cache)
    t = _upload(inp, dtype, cuda_device)
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G)
    outs = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], dirs, G)
    _check("h", from_torch(h), h_ref, dtype)
    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    for name, got, ref, ref_st in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), outs, g_ref, g_stored):
        got = from_torch(got)
        if dtype == "bf16" and name.startswith("dw"):
            record(test, name + " (unrounded h, not asserted: R18)", max(normwise(got[k], ref[k]) for k in
                                                                        range(got.shape[0])), TOL[dtype])
            _check(name + " (stored h)", got, ref_st, dtype)
        else:
            _check(name, got, ref, dtype)


def test_prenormalized_flag(cuda_device):
    """Pre-normalised taps with GSPN_FLAG_PRENORMALIZED == raw taps without it (fp32, normwise)."""
    import torch

    shape = (1, 3, 3, 20, 24, 0xF, "f32")
    cfg, inp, h_ref, _, _, _ = _oracle(shape, {})
    f = {k: v[1] for k, v in inp.items()}
    # normalise on the host with the oracle's convention by reading it through unit impulses is
    # overkill; use the definition: divide in-range taps by their sum (pinned in test_oracle).
    from tests import scan_views as sv
    D, G, H, W = 4, 3, 20, 24
    nl, nm, nr = np.zeros_like(f["w_l"]), np.zeros_like(f["w_m"]), np.zeros_like(f["w_r"])
    for k, d in enumerate(sv.DIR_ORDER):
        for g in range(G):
            wl, wm, wr = (sv.to_scan(f[n][k, 0, g], d) for n in ("w_l", "w_m", "w_r"))
            L, P = wm.shape
            a, b, c = np.zeros((L, P)), np.zeros((L, P)), np.zeros((L, P))
            for tt in range(L):
                M = sv.step_matrix(wl[tt], wm[tt], wr[tt])
                for r in range(P):
                    b[tt, r] = M[r, r]
                    a[tt, r] = M[r, r - 1] if r >= 1 else 0.0
                    c[tt, r] = M[r, r + 1] if r + 1 < P else 0.0
            nl[k, 0, g], nm[k, 0, g], nr[k, 0, g] = sv.from_scan(a, d), sv.from_scan(b, d), sv.from_scan(c, d)
    dev = cuda_device
    x = to_torch(inp["x"][0], "f32", dev)
    lam = to_torch(inp["lam"][0], "f32", dev)
    T = lambda a: torch.from_numpy(a.astype(np.float32)).to(dev)
    for flags in (gspn.FLAG_PRENORMALIZED, gspn.FLAG_PRENORMALIZED | gspn.FLAG_FORCE_GENERIC):
        h = gspn.fwd(x, T(nl), T(nm), T(nr), lam, 0xF, G, flags=flags)
        _check("h(prenorm)", from_torch(h), h_ref, "f32")


def test_fwd_deterministic_and_flip_symmetric(cuda_device):
    """fwd is bitwise deterministic; B2T(x) == flipH(T2B(flipH x)) and R2L == flipW(L2R(flipW)) bitwise."""
    import torch

    shape = (2, 4, 4, 48, 40, 0xF, "bf16")
    B, C, G, H, W, dirs, dtype = shape
    cfg = small_config(B, C, G, H, W, dirs, dtype, cfg_id=300)
    t = _upload(host_inputs(cfg), dtype, cuda_device)
    h1 = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G)
    h2 = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G)
    assert torch.equal(h1, h2)
    fh = lambda a: torch.flip(a, dims=[-2]).contiguous()
    fw = lambda a: torch.flip(a, dims=[-1]).contiguous()
    hb = gspn.fwd(fh(t["x"]), fh(t["w_l"][1:2]), fh(t["w_m"][1:2]), fh(t["w_r"][1:2]), fh(t["lam"][1:2]), 0x1, G)
    assert torch.equal(fh(hb)[0], h1[1])
    hr = gspn.fwd(fw(t["x"]), fw(t["w_l"][3:4]), fw(t["w_m"][3:4]), fw(t["w_r"][3:4]), fw(t["lam"][3:4]), 0x4, G)
    assert torch.equal(fw(hr)[0], h1[3])
