"""Test-side helpers (NOT the oracle, NOT the product): independent numpy restatements used to pin
the oracle — scan-coordinate views of a plane and the dense block operator G of Eq. 4.

Nothing here is imported by oracle/ or by the product package.
"""
from __future__ import annotations

import numpy as np

DIRS = {"T2B": 1, "B2T": 2, "L2R": 4, "R2L": 8}
DIR_ORDER = [1, 2, 4, 8]


def to_scan(plane: np.ndarray, d: int) -> np.ndarray:
    """[H, W] canonical plane -> [L, P] scan-coordinate view (gspn.h direction table)."""
    if d == 1:
        return plane
    if d == 2:
        return plane[::-1, :]
    if d == 4:
        return plane.T
    if d == 8:
        return plane[:, ::-1].T
    raise ValueError(d)


def from_scan(scan: np.ndarray, d: int) -> np.ndarray:
    if d == 1:
        return scan
    if d == 2:
        return scan[::-1, :]
    if d == 4:
        return scan.T
    if d == 8:
        return scan.T[:, ::-1]
    raise ValueError(d)


def step_matrix(wl_row, wm_row, wr_row) -> np.ndarray:
    """Row-stochastic tridiagonal step matrix D^-1 T of one step: T has w_m on the
    diagonal, w_l on the sub-diagonal (neighbour r-1) and w_r on the super-diagonal (neighbour r+1);
    entries that would fall outside the P x P matrix do not exist. D = diag(row sums of T)."""
    P = len(wm_row)
    T = np.diag(np.asarray(wm_row, dtype=np.float64))
    if P > 1:
        T += np.diag(np.asarray(wl_row[1:], dtype=np.float64), -1)
        T += np.diag(np.asarray(wr_row[:-1], dtype=np.float64), +1)
    return T / T.sum(axis=1, keepdims=True)


def dense_G(wl_s, wm_s, wr_s, lam_s) -> np.ndarray:
    """Eq. 4: H_v = G X_v with G_ij = (prod_{k=j+1..i} W_k) Lambda_j for j <= i,
    blocks P x P (reading R9). Inputs in scan coordinates [L, P]."""
    L, P = lam_s.shape
    Ws = [step_matrix(wl_s[t], wm_s[t], wr_s[t]) for t in range(L)]
    G = np.zeros((L * P, L * P))
    for i in range(L):
        for j in range(i + 1):
            M = np.eye(P)
            for k in range(j + 1, i + 1):
                M = Ws[k] @ M
            G[i * P:(i + 1) * P, j * P:(j + 1) * P] = M @ np.diag(lam_s[j])
    return G


def dense_forward_plane(x, wl, wm, wr, lam, d: int) -> np.ndarray:
    """h for one (direction, channel) plane via the dense operator (canonical [H, W] in and out)."""
    xs, ls = to_scan(x, d), to_scan(lam, d)
    G = dense_G(to_scan(wl, d), to_scan(wm, d), to_scan(wr, d), ls)
    hv = G @ xs.reshape(-1)
    return from_scan(hv.reshape(xs.shape), d)


def linear_attention_plane(x, wl, wm, wr, lam, d: int) -> np.ndarray:
    """PAPER.md:93 summation y_i = sum_{j<=i} (prod_{tau=j+1..i} w_tau) Lambda_j x_j with u = 1
    (upper limit read as j = i, reading R8)."""
    xs, ls = to_scan(x, d), to_scan(lam, d)
    wls, wms, wrs = to_scan(wl, d), to_scan(wm, d), to_scan(wr, d)
    L, P = xs.shape
    out = np.zeros((L, P))
    for i in range(L):
        acc = np.zeros(P)
        for j in range(i + 1):
            v = ls[j] * xs[j]
            for tau in range(j + 1, i + 1):
                v = step_matrix(wls[tau], wms[tau], wrs[tau]) @ v
            acc += v
        out[i] = acc
    return from_scan(out, d)
