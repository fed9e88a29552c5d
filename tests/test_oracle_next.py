"""Pins of the oracle's SURVEY §8(f) rows (CPU only; -m "not gpu"):

NEXT-1  output gate + direction merge, y = s * sum_d u_d (.) h_d (Eq. 2; the four passes
        "combined"; Sum / Mean) and its adjoint;
NEXT-2  GSPN-local ("splits each row or column into fixed-length segments of size kchunk
        and confines propagation to within those segments"; "at each kchunk segment start,
        h resets to 0"; a short last segment).

The kchunk pins do not re-type the reset rule: they compare the local scan with the GLOBAL scan run on
each segment's crop of the image (an independent construction of "confined to the segment"), plus the
kchunk = 1 / kchunk >= L special cases and finite differences. The merge pins use SPEC's 1x1 example,
the dense-connectivity property, bilinearity (dot test) and finite differences.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from tests.test_oracle import rand_inputs

ALL = 0xF
DIRS = (0x1, 0x2, 0x4, 0x8)


# ------------------------------------------------------------------------------------ NEXT-2 kchunk

@pytest.mark.parametrize("kchunk", [0, 7, 9, 100])
def test_kchunk_at_least_L_is_global(kchunk):
    rng = np.random.default_rng(1)
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 2, 2, 7, 5, ALL)
    ref = oracle.fwd(x, wl, wm, wr, lam, ALL, 2)
    # vertical L = 7, horizontal L = 5: kchunk >= 7 covers both
    got = oracle.fwd(x, wl, wm, wr, lam, ALL, 2, kchunk=kchunk)
    assert np.array_equal(got, ref)


def test_kchunk_one_isolates_every_step():
    """kchunk = 1: no step sees its predecessor, so h = lam x; the adjoint is local too."""
    rng = np.random.default_rng(2)
    x, wl, wm, wr, lam = rand_inputs(rng, 2, 3, 1, 4, 6, ALL)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1, kchunk=1)
    assert np.allclose(h, lam * x[None], rtol=0, atol=1e-15)
    dh = rng.uniform(-1, 1, h.shape)
    dx, dwl, dwm, dwr, dlam = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, 1, kchunk=1)
    assert np.allclose(dx, np.sum(dh * lam, axis=0), atol=1e-14)
    assert np.allclose(dlam, dh * x[None], atol=1e-15)
    for d in (dwl, dwm, dwr):
        assert np.all(d == 0.0)


def _segments(n, k):
    return [(s, min(s + k, n)) for s in range(0, n, k)]


@pytest.mark.parametrize("dirv", DIRS)
@pytest.mark.parametrize("kchunk", [2, 3, 4])
def test_kchunk_equals_global_scan_on_each_segment_crop(dirv, kchunk):
    """GSPN-local == the global scan applied to each segment's crop (rows for T2B/B2T, columns for
    L2R/R2L; segments fixed on the image grid, last one short: H = 7, W = 5), forward and backward."""
    rng = np.random.default_rng(10 + kchunk)
    B, C, G, H, W = 1, 2, 1, 7, 5
    x, wl, wm, wr, lam = rand_inputs(rng, B, C, G, H, W, dirv)
    dh = rng.uniform(-1, 1, lam.shape)
    h = oracle.fwd(x, wl, wm, wr, lam, dirv, G, kchunk=kchunk)
    grads = oracle.bwd(x, wl, wm, wr, lam, h, dh, dirv, G, kchunk=kchunk)
    vertical = dirv in (0x1, 0x2)
    n = H if vertical else W
    for lo, hi in _segments(n, kchunk):
        def crop(a):
            return a[..., lo:hi, :] if vertical else a[..., lo:hi]
        hc = oracle.fwd(crop(x), crop(wl), crop(wm), crop(wr), crop(lam), dirv, G)
        assert np.allclose(crop(h), hc, rtol=0, atol=1e-14), (lo, hi)
        gc = oracle.bwd(crop(x), crop(wl), crop(wm), crop(wr), crop(lam), hc, crop(dh), dirv, G)
        for name, a, b in zip(("dx", "dw_l", "dw_m", "dw_r", "dlam"), grads, gc):
            assert np.allclose(crop(a), b, rtol=0, atol=1e-13), (name, lo, hi)


def test_kchunk_backward_matches_finite_differences():
    rng = np.random.default_rng(5)
    B, C, G, H, W, k = 1, 2, 1, 5, 4, 2
    x, wl, wm, wr, lam = rand_inputs(rng, B, C, G, H, W, ALL)
    dh = rng.uniform(-1, 1, lam.shape)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, G, kchunk=k)
    grads = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, G, kchunk=k)
    inputs = [x, wl, wm, wr, lam]

    def loss():
        return float(np.sum(oracle.fwd(*inputs, ALL, G, kchunk=k) * dh))

    eps = 1e-6
    for gi, (arr, grad) in enumerate(zip(inputs, grads)):
        fd = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            old = arr[idx]
            arr[idx] = old + eps
            lp = loss()
            arr[idx] = old - eps
            lm = loss()
            arr[idx] = old
            fd[idx] = (lp - lm) / (2 * eps)
        err = np.abs(fd - grad).max() / max(np.abs(fd).max(), 1e-30)
        assert err < 1e-7, f"input {gi}: FD rel err {err}"


def test_kchunk_rejects_negative():
    rng = np.random.default_rng(6)
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 1, 1, 3, 3, 0x1)
    with pytest.raises(oracle.OracleError):
        oracle.fwd(x, wl, wm, wr, lam, 0x1, 1, kchunk=-1)


# ------------------------------------------------------------------------------------ NEXT-1 merge

def test_merge_one_by_one_image():
    """a 1x1 spatial input makes every scan a single step, so y = sum_d u_d lam_d x."""
    rng = np.random.default_rng(7)
    x, wl, wm, wr, lam = rand_inputs(rng, 2, 3, 3, 1, 1, ALL)
    u = rng.uniform(-1, 1, lam.shape)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 3)
    y = oracle.merge_fwd(h, u)
    assert np.allclose(y, (u[0] * lam[0] + u[1] * lam[1] + u[2] * lam[2] + u[3] * lam[3]) * x, atol=1e-15)
    assert np.allclose(oracle.merge_fwd(h, u, mean=True), y / 4, atol=1e-16)


def test_merge_identity_gate_single_direction():
    rng = np.random.default_rng(8)
    h = rng.uniform(-1, 1, (1, 2, 3, 4, 5))
    assert np.array_equal(oracle.merge_fwd(h, np.ones_like(h)), h[0])


def test_merge_dense_connectivity():
    """SPEC.md:506 ("dense pairwise connectivity"): 5x5, one channel, positive taps,
    lam = u = 1: after the four-direction merge every output depends on every input. Influence
    dy[p]/dx[q] read through the adjoint (merge_bwd then the scan's bwd) with dy = e_p."""
    rng = np.random.default_rng(9)
    H = W = 5
    x, wl, wm, wr, lam = rand_inputs(rng, 1, 1, 1, H, W, ALL)
    lam[:] = 1.0
    u = np.ones_like(lam)
    h = oracle.fwd(x, wl, wm, wr, lam, ALL, 1)
    infl = np.zeros((H * W, H * W))
    for p in range(H * W):
        dy = np.zeros((1, 1, H, W))
        dy.reshape(-1)[p] = 1.0
        dh, _ = oracle.merge_bwd(h, u, dy)
        dx = oracle.bwd(x, wl, wm, wr, lam, h, dh, ALL, 1)[0]
        infl[p] = dx.reshape(-1)
    assert np.all(np.abs(infl) > 1e-12)
    # one direction alone is NOT dense (T2B never reaches rows above): the merge is what connects
    dh1 = np.zeros_like(h)
    dh1[0, 0, 0, 0, 2] = 1.0  # output (0, 2) of T2B depends on row 0 only
    dx1 = oracle.bwd(x, wl, wm, wr, lam, h, dh1, ALL, 1)[0]
    assert np.all(dx1[0, 0, 1:] == 0.0)


@pytest.mark.parametrize("mean", [False, True])
def test_merge_adjoint_dot_test(mean):
    """y is bilinear in (h, u): <dy, y> = sum_d <dh_d, h_d> = sum_d <du_d, u_d>."""
    rng = np.random.default_rng(11)
    h = rng.uniform(-1, 1, (3, 2, 2, 4, 5))
    u = rng.uniform(-1, 1, h.shape)
    dy = rng.uniform(-1, 1, h.shape[1:])
    y = oracle.merge_fwd(h, u, mean)
    dh, du = oracle.merge_bwd(h, u, dy, mean)
    ref = float(np.sum(dy * y))
    assert abs(float(np.sum(dh * h)) - ref) < 1e-12
    assert abs(float(np.sum(du * u)) - ref) < 1e-12


def test_merge_backward_matches_finite_differences():
    rng = np.random.default_rng(12)
    h = rng.uniform(-1, 1, (4, 1, 2, 3, 3))
    u = rng.uniform(-1, 1, h.shape)
    dy = rng.uniform(-1, 1, h.shape[1:])
    dh, du = oracle.merge_bwd(h, u, dy, True)
    eps = 1e-6
    for arr, grad in ((h, dh), (u, du)):
        fd = np.zeros_like(arr)
        flat = arr.reshape(-1)
        for i in range(flat.size):
            old = flat[i]
            flat[i] = old + eps
            lp = float(np.sum(oracle.merge_fwd(h, u, True) * dy))
            flat[i] = old - eps
            lm = float(np.sum(oracle.merge_fwd(h, u, True) * dy))
            flat[i] = old
            fd.reshape(-1)[i] = (lp - lm) / (2 * eps)
        assert np.abs(fd - grad).max() < 1e-8


# ------------------------------------------------------------------------------------ NEXT-4 proxy

def test_proxy_identity_and_permutation():
    """M = I copies the channels; a permutation matrix permutes them (exact)."""
    rng = np.random.default_rng(13)
    x = rng.uniform(-1, 1, (2, 5, 3, 4))
    assert np.array_equal(oracle.proxy_mix(x, np.eye(5)), x)
    perm = [3, 0, 4, 1, 2]
    assert np.array_equal(oracle.proxy_mix(x, np.eye(5)[perm]), x[:, perm])


def test_proxy_matches_einsum_and_roundtrip():
    """Against numpy's einsum (a library primitive), and down-then-up with P_up = pinv(P_down) is the
    orthogonal projection onto the proxy subspace (idempotent; identity when C_proxy = C)."""
    rng = np.random.default_rng(14)
    x = rng.uniform(-1, 1, (3, 12, 5, 7))
    P = rng.normal(size=(4, 12))
    xp = oracle.proxy_mix(x, P)
    assert np.allclose(xp, np.einsum("pc,bchw->bphw", P, x), atol=1e-12)
    Q = np.linalg.pinv(P)
    y = oracle.proxy_mix(xp, Q)
    assert np.allclose(oracle.proxy_mix(oracle.proxy_mix(y, P), Q), y, atol=1e-10)
    Pf = rng.normal(size=(12, 12))
    assert np.allclose(oracle.proxy_mix(oracle.proxy_mix(x, Pf), np.linalg.inv(Pf)), x, atol=1e-9)


def test_proxy_adjoint_and_weight_gradient():
    """<dout, M x> = <M^T dout, x> = <dM, M> with dM = wgrad(dout, x); finite differences on M."""
    rng = np.random.default_rng(15)
    x = rng.uniform(-1, 1, (2, 6, 3, 5))
    M = rng.normal(size=(3, 6))
    dout = rng.uniform(-1, 1, (2, 3, 3, 5))
    ref = float(np.sum(dout * oracle.proxy_mix(x, M)))
    assert abs(float(np.sum(oracle.proxy_mix(dout, M.T) * x)) - ref) < 1e-12
    dM = oracle.proxy_wgrad(dout, x)
    assert abs(float(np.sum(dM * M)) - ref) < 1e-12
    eps = 1e-6
    fd = np.zeros_like(M)
    for idx in np.ndindex(M.shape):
        Mp, Mm = M.copy(), M.copy()
        Mp[idx] += eps
        Mm[idx] -= eps
        fd[idx] = (np.sum(dout * oracle.proxy_mix(x, Mp)) - np.sum(dout * oracle.proxy_mix(x, Mm))) / (2 * eps)
    assert np.abs(fd - dM).max() < 1e-8


def test_compact_block_linear_attention_rank():
    """The compact block: down-project, scan with one shared affinity (G = 1), up-project.
    With lam = 1 it is linear in x with rank <= C_proxy per pixel pair -- the low-rank structure of
    PAPER.md:644 ('analogous to low-rank matrix factorization')."""
    rng = np.random.default_rng(16)
    B, C, Cp, H, W = 1, 6, 2, 3, 3
    P = rng.normal(size=(Cp, C))
    Q = rng.normal(size=(C, Cp))
    wl, wm, wr = (rng.uniform(0.05, 1, (4, B, 1, H, W)) for _ in range(3))
    lam = np.ones((4, B, Cp, H, W))

    def block(x):
        h = oracle.fwd(oracle.proxy_mix(x, P), wl, wm, wr, lam, 0xF, 1)
        return oracle.proxy_mix(h.sum(axis=0), Q)

    # Jacobian block between input pixel q and output pixel p is C x C of rank <= Cp
    cols = []
    for k in range(C * H * W):
        e = np.zeros(C * H * W)
        e[k] = 1.0
        cols.append(block(e.reshape(B, C, H, W)).reshape(-1))
    J = np.array(cols).T.reshape(C, H * W, C, H * W)
    for p_ in range(H * W):
        for q in range(H * W):
            assert np.linalg.matrix_rank(J[:, p_, :, q], tol=1e-9) <= Cp
