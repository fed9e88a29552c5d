"""Pins of the fp64 oracle against things other than itself (CPU only; -m "not gpu").

Each pin would fail on a plausible mistake: a dropped term (cumsum / constant-input closed forms,
dense G), a wrong sign or index (finite differences, dot test, Euler identity), a transposed operand
or direction (dense G per direction, flip/transpose symmetry), a wrong boundary rule (golden taps,
constant input incl. edges), a wrong group sum (grouped == sum of per-channel with shared taps).
"""
from __future__ import annotations

import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests import scan_views as sv

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ALL = 0xF


def rand_inputs(rng, B, C, G, H, W, dirs, wlo=0.05):
    D = bin(dirs).count("1")
    x = rng.uniform(-1, 1, (B, C, H, W))
    wl = rng.uniform(wlo, 1, (D, B, G, H, W))
    wm = rng.uniform(wlo, 1, (D, B, G, H, W))
    wr = rng.uniform(wlo, 1, (D, B, G, H, W))
    lam = rng.uniform(0, 1, (D, B, C, H, W))
    return x, wl, wm, wr, lam


def dir_list(dirs):
    return [d for d in sv.DIR_ORDER if dirs & d]


# ---------------------------------------------------------------- golden fixtures (SPEC examples)

def _read_golden_taps():
    rows = []
    with open(os.path.join(GOLDEN, "normalisation_taps.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            P, r, wl, wm, wr, a, b, c = line.split()
            rows.append((int(P), int(r), float(wl), float(wm), float(wr),
                         float(Fraction(a)), float(Fraction(b)), float(Fraction(c))))
    return rows


@pytest.mark.parametrize("row", _read_golden_taps())
def test_golden_normalised_taps(row):
    """Read the normalised taps out of the oracle with impulses: T2B, H = 2, lambda = 1, x row 0 = e_k,
    row 1 = 0  =>  h_1[r] = a[r] [k = r-1] + b[r] [k = r] + c[r] [k = r+1]."""
    P, r, wl, wm, wr, a, b, c = row
    got = {}
    for k, name in ((r - 1, "a"), (r, "b"), (r + 1, "c")):
        if k < 0 or k >= P:
            got[name] = 0.0
            continue
        x = np.zeros((1, 1, 2, P))
        x[0, 0, 0, k] = 1.0
        lam = np.ones((1, 1, 1, 2, P))
        Wl = np.full((1, 1, 1, 2, P), 0.5)
        Wm = np.full((1, 1, 1, 2, P), 0.5)
        Wr = np.full((1, 1, 1, 2, P), 0.5)
        Wl[0, 0, 0, 1, r], Wm[0, 0, 0, 1, r], Wr[0, 0, 0, 1, r] = wl, wm, wr
        h = oracle.fwd(x, Wl, Wm, Wr, lam, 1, 1)
        got[name] = h[0, 0, 0, 1, r]
    np.testing.assert_allclose([got["a"], got["b"], got["c"]], [a, b, c], rtol=0, atol=1e-15)


def test_golden_spec_2x2_t2b():
    xs, hs = [], []
    with open(os.path.join(GOLDEN, "spec_2x2_t2b.txt")) as f:
        for line in f:
            if line.startswith("x "):
                xs.append([float(v) for v in line.split()[1:]])
            elif line.startswith("h "):
                hs.append([float(v) for v in line.split()[1:]])
    x = np.array(xs)[None, None]
    ones = np.ones((1, 1, 1, 2, 2))
    h = oracle.fwd(x, ones, ones, ones, ones, 1, 1)
    np.testing.assert_array_equal(h[0, 0, 0], np.array(hs))


# ---------------------------------------------------------------- dense operator G (Eq. 4) and Eq. 1 sum

@pytest.mark.parametrize("H,W", [(1, 1), (1, 5), (4, 1), (3, 4), (5, 3), (6, 6), (8, 7)])
def test_forward_equals_dense_G(H, W):
    rng = np.random.default_rng(100 + 10 * H + W)
    B, C, G = 2, 3, 3
    x, wl, wm, wr, lam = rand_inputs(rng, B, C, G, H, W, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, G)
    for k, d in enumerate(dir_list(ALL)):
        for b in range(B):
            for c in range(C):
                ref = sv.dense_forward_plane(x[b, c], wl[k, b, c], wm[k, b, c], wr[k, b, c], lam[k, b, c], d)
                np.testing.assert_allclose(h[k, b, c], ref, rtol=0, atol=1e-14)


def test_forward_grouped_equals_dense_G_shared_w():
    """Eq. 3: one w_i shared by the channels of a group (G = 1 and G = 2 of C = 4)."""
    rng = np.random.default_rng(7)
    for G in (1, 2):
        B, C, H, W = 2, 4, 5, 6
        x, wl, wm, wr, lam = rand_inputs(rng, B, C, G, H, W, ALL)
        h = oracle.fwd(x, wl, wm, wr, lam, ALL, G)
        Cg = C // G
        for k, d in enumerate(dir_list(ALL)):
            for b in range(B):
                for c in range(C):
                    g = c // Cg
                    ref = sv.dense_forward_plane(x[b, c], wl[k, b, g], wm[k, b, g], wr[k, b, g], lam[k, b, c], d)
                    np.testing.assert_allclose(h[k, b, c], ref, rtol=0, atol=1e-14)


def test_dense_G_blocks_row_stochastic():
    """With lambda = 1 every block row of G applied to a constant input gives (t+1): blocks are
    row-stochastic. Checked on the oracle output: constant x = 1 -> h_t = t + 1."""
    rng = np.random.default_rng(3)
    H, W = 7, 9
    _, wl, wm, wr, _ = rand_inputs(rng, 1, 1, 1, H, W, ALL)
    x = np.ones((1, 1, H, W))
    lam = np.ones((4, 1, 1, H, W))
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    for k, d in enumerate(dir_list(ALL)):
        hs = sv.to_scan(h[k, 0, 0], d)
        L = hs.shape[0]
        np.testing.assert_allclose(hs, np.repeat(np.arange(1, L + 1, dtype=float)[:, None], hs.shape[1], 1),
                                   rtol=0, atol=1e-13)


def test_linear_attention_form():
    rng = np.random.default_rng(11)
    H, W = 4, 5
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 1, 1, H, W, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    for k, d in enumerate(dir_list(ALL)):
        ref = sv.linear_attention_plane(x[0, 0], wl[k, 0, 0], wm[k, 0, 0], wr[k, 0, 0], lam[k, 0, 0], d)
        np.testing.assert_allclose(h[k, 0, 0], ref, rtol=0, atol=1e-14)


# ---------------------------------------------------------------- closed forms

def test_cumsum_when_side_taps_zero():
    """w_l = w_r = 0, any w_m > 0 -> h = cumulative sum of lambda x along the scan (BASELINE north_star)."""
    rng = np.random.default_rng(5)
    H, W = 6, 7
    x, _, wm, _, lam = rand_inputs(rng, 2, 2, 2, H, W, ALL)
    z = np.zeros_like(wm)
    h = oracle.fwd(x, z, wm, z, lam, ALL, 2)
    for k, d in enumerate(dir_list(ALL)):
        for b in range(2):
            for c in range(2):
                ref = np.cumsum(sv.to_scan(lam[k, b, c] * x[b, c], d), axis=0)
                np.testing.assert_allclose(sv.to_scan(h[k, b, c], d), ref, rtol=0, atol=1e-14)


def test_width_one_is_cumsum():
    rng = np.random.default_rng(6)
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 1, 1, 9, 1, 0x3)
    h = oracle.fwd(x, wl, wm, wr, lam, 0x3, 1)
    np.testing.assert_allclose(h[0, 0, 0, :, 0], np.cumsum(lam[0, 0, 0, :, 0] * x[0, 0, :, 0]), atol=1e-15)
    np.testing.assert_allclose(h[1, 0, 0, ::-1, 0], np.cumsum((lam[1, 0, 0] * x[0, 0])[::-1, 0]), atol=1e-15)


def test_length_one_is_lambda_x():
    rng = np.random.default_rng(8)
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 1, 1, 6, 0x3)
    h = oracle.fwd(x, wl, wm, wr, lam, 0x3, 1)
    for k in range(2):
        np.testing.assert_array_equal(h[k], lam[k] * x)


def test_constant_input_grows_linearly_incl_edges():
    """Constant lambda x = k -> h_t = (t+1) k at EVERY r, including r = 0 and r = P-1. Zero-padding h
    instead of dropping the out-of-range taps (reading R2) would break the edges."""
    rng = np.random.default_rng(9)
    H, W = 5, 8
    _, wl, wm, wr, _ = rand_inputs(rng, 1, 1, 1, H, W, ALL)
    x = np.full((1, 1, H, W), 0.75)
    lam = np.full((4, 1, 1, H, W), 2.0)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    for k, d in enumerate(dir_list(ALL)):
        hs = sv.to_scan(h[k, 0, 0], d)
        for t in range(hs.shape[0]):
            np.testing.assert_allclose(hs[t], 1.5 * (t + 1), rtol=1e-14)


def test_impulse_at_first_step_propagates_constant():
    """lambda x = k at t = 0 only -> h_t = k for all t (row-stochastic propagation of a constant)."""
    rng = np.random.default_rng(10)
    H, W = 6, 6
    _, wl, wm, wr, _ = rand_inputs(rng, 1, 1, 1, H, W, ALL)
    x = np.full((1, 1, H, W), -0.3)
    for k, d in enumerate(dir_list(ALL)):
        lam_s = np.zeros((H, W))
        lam_s[0, :] = 1.0  # scan step 0 (square plane so the scan view is H x W)
        lam = np.zeros((4, 1, 1, H, W))
        lam[k, 0, 0] = sv.from_scan(lam_s, d)
        h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
        np.testing.assert_allclose(h[k, 0, 0], -0.3, rtol=1e-14)


def test_prenormalized_flag_matches_raw():
    rng = np.random.default_rng(12)
    H, W = 5, 6
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 2, H, W, ALL)
    h_raw = oracle.fwd(x, wl, wm, wr, lam, ALL, 2)
    nl, nm, nr = np.zeros_like(wl), np.zeros_like(wm), np.zeros_like(wr)
    for k, d in enumerate(dir_list(ALL)):
        for g in range(2):
            L, P = sv.to_scan(wm[k, 0, g], d).shape
            a = np.zeros((L, P)); b = np.zeros((L, P)); c = np.zeros((L, P))
            wls, wms, wrs = sv.to_scan(wl[k, 0, g], d), sv.to_scan(wm[k, 0, g], d), sv.to_scan(wr[k, 0, g], d)
            for t in range(L):
                M = sv.step_matrix(wls[t], wms[t], wrs[t])
                for r in range(P):
                    b[t, r] = M[r, r]
                    if r >= 1:
                        a[t, r] = M[r, r - 1]
                    if r + 1 < P:
                        c[t, r] = M[r, r + 1]
            nl[k, 0, g], nm[k, 0, g], nr[k, 0, g] = sv.from_scan(a, d), sv.from_scan(b, d), sv.from_scan(c, d)
    h_pre = oracle.fwd(x, nl, nm, nr, lam, ALL, 2, flags=oracle.PRENORMALIZED)
    np.testing.assert_allclose(h_pre, h_raw, rtol=0, atol=1e-14)


def test_stability_bound():
    """||h_t||_inf <= ||h_{t-1}||_inf + ||lambda_t x_t||_inf."""
    rng = np.random.default_rng(13)
    H, W = 16, 12
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 1, 1, H, W, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    for k, d in enumerate(dir_list(ALL)):
        hs, src = sv.to_scan(h[k, 0, 0], d), sv.to_scan(lam[k, 0, 0] * x[0, 0], d)
        for t in range(1, hs.shape[0]):
            assert np.abs(hs[t]).max() <= np.abs(hs[t - 1]).max() + np.abs(src[t]).max() + 1e-15


def test_nonpositive_row_sum_rejected():
    x = np.ones((1, 1, 2, 3))
    z = np.zeros((1, 1, 1, 2, 3))
    with pytest.raises(oracle.OracleError):
        oracle.fwd(x, z, z, z, np.ones((1, 1, 1, 2, 3)), 1, 1)


# ---------------------------------------------------------------- direction symmetry (bitwise)

def test_direction_flip_transpose_symmetry():
    rng = np.random.default_rng(14)
    H, W = 5, 7
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 1, 1, H, W, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    # B2T(x) = flipH(T2B(flipH(x)))   (taps flipped with the plane; w_l stays the smaller column)
    f = lambda a: a[..., ::-1, :].copy()
    hb = oracle.fwd(f(x), f(wl[1:2]), f(wm[1:2]), f(wr[1:2]), f(lam[1:2]), 0x1, 1)
    np.testing.assert_array_equal(f(hb[0]), h[1])
    # R2L(x) = flipW(L2R(flipW(x)))
    g = lambda a: a[..., :, ::-1].copy()
    hr = oracle.fwd(g(x), g(wl[3:4]), g(wm[3:4]), g(wr[3:4]), g(lam[3:4]), 0x4, 1)
    np.testing.assert_array_equal(g(hr[0]), h[3])
    # L2R(x) = T2B(x^T)^T   (w_l = smaller row index = smaller column index after transpose)
    tr = lambda a: np.swapaxes(a, -1, -2).copy()
    ht = oracle.fwd(tr(x), tr(wl[2:3]), tr(wm[2:3]), tr(wr[2:3]), tr(lam[2:3]), 0x1, 1)
    np.testing.assert_array_equal(tr(ht[0]), h[2])


# ---------------------------------------------------------------- backward

def _loss(x, wl, wm, wr, lam, dh, dirs, G):
    return float(np.sum(oracle.fwd(x, wl, wm, wr, lam, dirs, G) * dh))


@pytest.mark.parametrize("G", [3, 1])
def test_backward_matches_finite_differences(G):
    rng = np.random.default_rng(20 + G)
    B, C, H, W = 1, 3, 4, 5
    x, wl, wm, wr, lam = rand_inputs(rng, B, C, G, H, W, ALL)
    dh = rng.uniform(-1, 1, lam.shape)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, G)
    grads = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, G)
    inputs = [x, wl, wm, wr, lam]
    eps = 1e-6
    for gi, (arr, grad) in enumerate(zip(inputs, [grads[0], grads[1], grads[2], grads[3], grads[4]])):
        fd = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            old = arr[idx]
            arr[idx] = old + eps
            lp = _loss(*inputs, dh, ALL, G)
            arr[idx] = old - eps
            lm = _loss(*inputs, dh, ALL, G)
            arr[idx] = old
            fd[idx] = (lp - lm) / (2 * eps)
        err = np.abs(fd - grad).max() / max(np.abs(fd).max(), 1e-30)
        assert err < 1e-7, f"input {gi}: FD rel err {err}"


def test_backward_zero_upstream_gives_zero():
    rng = np.random.default_rng(30)
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 1, 4, 4, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    for gr in oracle.bwd(x, wl, wm, wr, lam, h, np.zeros_like(h), ALL, 1):
        assert not np.any(gr)


def test_backward_length_one_chain_rule():
    """L = 1: dlam = dh x, dx = sum_d dh lam, dw = 0 (SPEC.md:200 with u = 1)."""
    rng = np.random.default_rng(31)
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 2, 1, 5, 0x3)
    h = oracle.fwd(x, wl, wm, wr, lam, 0x3, 2)
    dh = rng.uniform(-1, 1, h.shape)
    dx, dwl, dwm, dwr, dlam = oracle.bwd(x, wl, wm, wr, lam, h, dh, 0x3, 2)
    np.testing.assert_allclose(dlam, dh * x[None], atol=1e-15)
    np.testing.assert_allclose(dx, (dh * lam).sum(0), atol=1e-15)
    assert not np.any(dwl) and not np.any(dwm) and not np.any(dwr)


def test_adjoint_dot_and_euler_identities():
    """h is linear in x and in lambda: <dh, h> = <dx, x> = sum <dlam, lam>. h is degree-0 homogeneous
    in the raw taps of a pixel: w_l dw_l + w_m dw_m + w_r dw_r = 0 at every pixel."""
    rng = np.random.default_rng(32)
    x, wl, wm, wr, lam = rand_inputs(rng, 2, 4, 2, 6, 5, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 2)
    dh = rng.uniform(-1, 1, h.shape)
    dx, dwl, dwm, dwr, dlam = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, 2)
    a = np.sum(dh * h)
    np.testing.assert_allclose(np.sum(dx * x), a, rtol=1e-12)
    np.testing.assert_allclose(np.sum(dlam * lam), a, rtol=1e-12)
    np.testing.assert_allclose(wl * dwl + wm * dwm + wr * dwr, 0.0, atol=1e-13)


def test_adjoint_mass_conservation():
    """lambda = 1, dh = unit impulse at the last step at one position -> sum_r g_t[r] = 1 for all t;
    with x = 1, dlam = g, so every scan row of dlam sums to 1 (the transpose of a row-stochastic map
    preserves mass)."""
    rng = np.random.default_rng(33)
    H, W = 6, 7
    _, wl, wm, wr, _ = rand_inputs(rng, 1, 1, 1, H, W, ALL)
    x = np.ones((1, 1, H, W))
    lam = np.ones((4, 1, 1, H, W))
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    dh = np.zeros_like(h)
    for k, d in enumerate(dir_list(ALL)):
        s = np.zeros(sv.to_scan(np.zeros((H, W)), d).shape)
        s[-1, s.shape[1] // 2] = 1.0
        dh[k, 0, 0] = sv.from_scan(s, d)
    _, _, _, _, dlam = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, 1)
    for k, d in enumerate(dir_list(ALL)):
        np.testing.assert_allclose(sv.to_scan(dlam[k, 0, 0], d).sum(axis=1), 1.0, rtol=1e-13)


def test_grouped_dw_is_channel_sum_of_per_channel():
    """G = 1 over C channels == per-channel (G = C) run with the shared taps replicated, dw summed
    over channels (the Jacobian of the normalisation is linear in the tap gradients)."""
    rng = np.random.default_rng(34)
    B, C, H, W = 2, 3, 4, 6
    x, wl, wm, wr, lam = rand_inputs(rng, B, C, 1, H, W, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    dh = rng.uniform(-1, 1, h.shape)
    g1 = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, 1)
    rep = lambda a: np.repeat(a, C, axis=2)
    hC = oracle.fwd(x, rep(wl), rep(wm), rep(wr), lam, ALL, C)
    np.testing.assert_array_equal(hC, h)
    gC = oracle.bwd(x, rep(wl), rep(wm), rep(wr), lam, hC, dh, ALL, C)
    np.testing.assert_allclose(gC[0], g1[0], atol=1e-14)
    np.testing.assert_allclose(gC[4], g1[4], atol=1e-14)
    for k in (1, 2, 3):
        np.testing.assert_allclose(gC[k].sum(axis=2, keepdims=True), g1[k], atol=1e-13)


def test_threads_do_not_change_results():
    rng = np.random.default_rng(35)
    x, wl, wm, wr, lam = rand_inputs(rng, 3, 4, 2, 7, 6, ALL)
    h1 = oracle.fwd(x, wl, wm, wr, lam, ALL, 2, threads=1)
    h4 = oracle.fwd(x, wl, wm, wr, lam, ALL, 2, threads=4)
    np.testing.assert_array_equal(h1, h4)
    dh = rng.uniform(-1, 1, h1.shape)
    for a, b in zip(oracle.bwd(x, wl, wm, wr, lam, h1, dh, ALL, 2, threads=1),
                    oracle.bwd(x, wl, wm, wr, lam, h1, dh, ALL, 2, threads=3)):
        np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- backward under GSPN_FLAG_PRENORMALIZED

def _loss_flags(x, wl, wm, wr, lam, dh, dirs, G, flags):
    return float(np.sum(oracle.fwd(x, wl, wm, wr, lam, dirs, G, flags=flags) * dh))


@pytest.mark.parametrize("G", [3, 1])
@pytest.mark.parametrize("dirs", [0x1, 0x2, 0x4, 0x8])
def test_backward_prenormalized_matches_finite_differences(G, dirs):
    """PRENORMALIZED (R1): the taps act as given, out-of-range ones dropped, so dw = (Da, Db, Dc) masked
    at the chain ends and zero at t = 0. Pinned against central differences of the (separately pinned,
    test_prenormalized_flag_matches_raw) prenormalised forward, per direction, G = C and G = 1. Taps
    are drawn unnormalised (row sums != 1) so a Jacobian applied by mistake would show."""
    rng = np.random.default_rng(40 + G + 7 * dirs)
    B, C, H, W = 1, 3, 4, 5
    x, wl, wm, wr, lam = rand_inputs(rng, B, C, G, H, W, dirs)
    dh = rng.uniform(-1, 1, lam.shape)
    F = oracle.PRENORMALIZED
    h = oracle.fwd(x, wl, wm, wr, lam, dirs, G, flags=F)
    grads = oracle.bwd(x, wl, wm, wr, lam, h, dh, dirs, G, flags=F)
    inputs = [x, wl, wm, wr, lam]
    eps = 1e-6
    for gi, (arr, grad) in enumerate(zip(inputs, grads)):
        fd = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            old = arr[idx]
            arr[idx] = old + eps
            lp = _loss_flags(*inputs, dh, dirs, G, F)
            arr[idx] = old - eps
            lm = _loss_flags(*inputs, dh, dirs, G, F)
            arr[idx] = old
            fd[idx] = (lp - lm) / (2 * eps)
        err = np.abs(fd - grad).max() / max(np.abs(fd).max(), 1e-30)
        assert err < 1e-7, f"dirs {dirs:#x} input {gi}: FD rel err {err}"


def test_backward_prenormalized_out_of_range_taps_are_zero():
    """The taps that fall off the chain (w_l at r = 0, w_r at r = P-1) and every tap of step 0 (h_{-1} = 0)
    reach nothing, so their gradient is exactly 0 -- also when the flag skips the normalisation."""
    rng = np.random.default_rng(46)
    H, W = 5, 6
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 1, H, W, ALL)
    F = oracle.PRENORMALIZED
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1, flags=F)
    dh = rng.uniform(-1, 1, h.shape)
    _, dwl, dwm, dwr, _ = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, 1, flags=F)
    for k, d in enumerate(dir_list(ALL)):
        a, b, c = (sv.to_scan(t[k, 0, 0], d) for t in (dwl, dwm, dwr))
        assert not np.any(a[:, 0]) and not np.any(c[:, -1])
        assert not np.any(a[0]) and not np.any(b[0]) and not np.any(c[0])
        assert np.all(np.abs(b[1:]) > 0)


def test_backward_prenormalized_length_one_and_zero_upstream():
    rng = np.random.default_rng(47)
    F = oracle.PRENORMALIZED
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 2, 1, 5, 0x3)
    h = oracle.fwd(x, wl, wm, wr, lam, 0x3, 2, flags=F)
    dh = rng.uniform(-1, 1, h.shape)
    dx, dwl, dwm, dwr, dlam = oracle.bwd(x, wl, wm, wr, lam, h, dh, 0x3, 2, flags=F)
    np.testing.assert_allclose(dlam, dh * x[None], atol=1e-15)
    np.testing.assert_allclose(dx, (dh * lam).sum(0), atol=1e-15)
    assert not np.any(dwl) and not np.any(dwm) and not np.any(dwr)
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 1, 4, 4, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1, flags=F)
    for gr in oracle.bwd(x, wl, wm, wr, lam, h, np.zeros_like(h), ALL, 1, flags=F):
        assert not np.any(gr)


def test_backward_prenormalized_equals_raw_chain_rule():
    """Raw-tap gradients = the prenormalised gradients pushed through the normalisation Jacobian:
    dw_k = (Dn_k - sum_j n_j Dn_j) / S, with n the normalised taps and Dn the PRENORMALIZED dw evaluated at
    n. A second, independent route to the raw branch through the prenormalised one."""
    rng = np.random.default_rng(48)
    H, W = 4, 6
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 2, H, W, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 2)
    dh = rng.uniform(-1, 1, h.shape)
    raw = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, 2)
    nl, nm, nr, S = (np.zeros_like(wl) for _ in range(4))
    for k, d in enumerate(dir_list(ALL)):
        for g in range(2):
            a, b, c = (sv.to_scan(t[k, 0, g], d).copy() for t in (wl, wm, wr))
            a[:, 0] = 0.0
            c[:, -1] = 0.0
            s = a + b + c
            nl[k, 0, g], nm[k, 0, g], nr[k, 0, g] = (sv.from_scan(t / s, d) for t in (a, b, c))
            S[k, 0, g] = sv.from_scan(s, d)
    pre = oracle.bwd(x, nl, nm, nr, lam, h, dh, ALL, 2, flags=oracle.PRENORMALIZED)
    np.testing.assert_allclose(pre[0], raw[0], atol=1e-13)
    np.testing.assert_allclose(pre[4], raw[4], atol=1e-13)
    q = nl * pre[1] + nm * pre[2] + nr * pre[3]
    for k, (Dn, n) in enumerate(zip(pre[1:4], (nl, nm, nr))):
        ref = (Dn - q) / S
        if k == 0:
            ref = np.where(nl == 0, 0.0, ref)
        if k == 2:
            ref = np.where(nr == 0, 0.0, ref)
        np.testing.assert_allclose(raw[1 + k], ref, atol=1e-13)


def test_oracle_cli_runs_config1():
    """The stand-alone oracle CLI (python -m oracle) runs BASELINE config 1 end to end."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "oracle", "--config", "1", "--threads", "2"], capture_output=True,
                         text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr
    assert "config 1" in out.stdout and "dlam" in out.stdout
