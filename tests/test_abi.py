"""C ABI: the library loads on a CPU-only box, exports every symbol include/gspn.h declares, and every
validation error path returns the right status before any CUDA call (no device needed)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

import paper_2512_07884_b200 as gspn
from paper_2512_07884_b200.build import LIBGSPN, ROOT

HEADER = os.path.join(ROOT, "include", "gspn.h")
A = 0x10000  # fake, 16-byte aligned, never dereferenced (validation fails first)


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(gspn_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert {"gspn_fwd", "gspn_bwd", "gspn_bwd_workspace_bytes", "gspn_status_string",
            "gspn_last_error_detail", "gspn_algorithmic_bytes"} <= set(names)
    out = subprocess.check_output(["nm", "-D", "--defined-only", LIBGSPN]).decode()
    exported = set(re.findall(r"\bT (gspn_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    L = gspn.lib()
    for n in names:
        assert hasattr(L, n)


def fwd_call(**kw):
    a = dict(x=A, wl=A, wm=A, wr=A, lam=A, h=A + (1 << 30), B=1, C=4, H=8, W=8, dirs=0xF, G=4, dt=1, flags=0)
    a.update(kw)
    return gspn.lib().gspn_fwd(a["x"], a["wl"], a["wm"], a["wr"], a["lam"], a["h"], a["B"], a["C"], a["H"], a["W"],
                               a["dirs"], a["G"], a["dt"], a["flags"], None)


def detail():
    return gspn.lib().gspn_last_error_detail().decode()


@pytest.mark.parametrize("kw,needle", [
    (dict(x=None), "x is NULL"),
    (dict(lam=None), "lam is NULL"),
    (dict(h=None), "h is NULL"),
    (dict(wm=A + 8), "w_m is not 16-byte aligned"),
    (dict(B=0), "B must be"),
    (dict(C=-1), "C must be"),
    (dict(H=0), "H must be"),
    (dict(W=0), "W must be"),
    (dict(G=0), "groups must be"),
    (dict(G=3), "C % groups"),
    (dict(dirs=0), "dirs"),
    (dict(dirs=16), "dirs"),
    (dict(flags=0x80), "flags"),
    (dict(dt=7), "dtype"),
])
def test_fwd_validation(kw, needle):
    assert fwd_call(**kw) == 1
    assert needle in detail()


def test_fwd_aliasing_rejected():
    # h overlaps lam
    assert fwd_call(lam=A + (1 << 20), h=A + (1 << 20) + 1024) == 1
    assert "overlaps" in detail()


def bwd_call(ws=A + (40 << 30), ws_bytes=1 << 40, flags=0, groups=2, **kw):
    base = 1 << 30
    p = dict(x=A, wl=A + base, wm=A + 2 * base, wr=A + 3 * base, lam=A + 4 * base, h=A + 5 * base,
             dh=A + 6 * base, dx=A + 7 * base, dwl=A + 8 * base, dwm=A + 9 * base, dwr=A + 10 * base,
             dlam=A + 11 * base)
    p.update(kw)
    return gspn.lib().gspn_bwd(p["x"], p["wl"], p["wm"], p["wr"], p["lam"], p["h"], p["dh"], p["dx"], p["dwl"],
                               p["dwm"], p["dwr"], p["dlam"], 2, 4, 16, 16, 0xF, groups, 1, flags, ws, ws_bytes, None)


def test_bwd_validation():
    assert bwd_call(dh=None) == 1 and "dh is NULL" in detail()
    assert bwd_call(dlam=A + 3) == 1 and "dlam is not 16-byte aligned" in detail()
    assert bwd_call(ws=None) == 1 and "workspace is NULL" in detail()
    assert bwd_call(ws_bytes=16) == 1 and "workspace too small" in detail()
    assert bwd_call(dx=A + 4 * (1 << 30)) == 1 and "overlaps" in detail()  # dx on lam
    assert bwd_call(dwm=A + 8 * (1 << 30)) == 1 and "overlaps" in detail()  # dw_m on dw_l
    assert bwd_call(flags=0x40) == 1 and "unknown bits" in detail()


def test_dw_f32_flag_validation():
    """GSPN_FLAG_DW_F32: fp32 dw partial sums, grouped weights only; the dw spans are sized in fp32."""
    assert bwd_call(flags=0x20, groups=4) == 2 and "DW_F32" in detail()  # groups == C: unsupported
    # bf16 dw of [4,2,2,16,16] = 4 KB would fit between dw_l and dw_m 6 KB apart; fp32 (8 KB) overlaps
    assert bwd_call(flags=0x20, dwm=A + 8 * (1 << 30) + 6144) == 1 and "overlaps" in detail()


def test_workspace_and_bytes():
    L = gspn.lib()
    assert L.gspn_bwd_workspace_bytes(4, 320, 512, 512, 0xF, 320, 1) > 0
    assert L.gspn_bwd_workspace_bytes(4, 320, 512, 512, 0xF, 3, 1) == 0  # invalid groups
    # config 4 fwd+bwd = 42,278.58 MB, fwd = s[N(1+2D) + 3 D N_w]
    f = L.gspn_algorithmic_bytes(4, 320, 512, 512, 0xF, 320, 1, 0)
    b = L.gspn_algorithmic_bytes(4, 320, 512, 512, 0xF, 320, 1, 1)
    assert abs((f + b) / 1e6 - 42278.58) < 0.01
    assert b == 2 * f
    # config 5 (G = 1): 9,361.69 MB
    f5 = L.gspn_algorithmic_bytes(1, 40, 2048, 2048, 0xF, 1, 1, 0)
    assert abs(3 * f5 / 1e6 - 9361.69) < 0.01


def test_status_strings():
    L = gspn.lib()
    assert L.gspn_status_string(0) == b"GSPN_OK"
    assert L.gspn_status_string(2) == b"GSPN_ERR_UNSUPPORTED"


def test_python_binding_refuses_cpu_tensors():
    torch = pytest.importorskip("torch")
    x = torch.zeros(1, 2, 4, 4)
    w = torch.ones(1, 1, 2, 4, 4)
    lam = torch.ones(1, 1, 2, 4, 4)
    with pytest.raises(ValueError, match="CUDA tensor"):
        gspn.fwd(x, w, w, w, lam, dirs=1, groups=2)


def test_local_validation():
    """gspn_fwd_local / gspn_bwd_local (GSPN-local) reject a negative kchunk before any CUDA call
    and otherwise validate exactly like gspn_fwd / gspn_bwd."""
    L = gspn.lib()
    base = 1 << 30
    assert L.gspn_fwd_local(A, A, A, A, A, A + base, 1, 4, 8, 8, 0xF, 4, -1, 1, 0, None) == 1
    assert "kchunk" in detail()
    assert L.gspn_fwd_local(None, A, A, A, A, A + base, 1, 4, 8, 8, 0xF, 4, 2, 1, 0, None) == 1
    assert "x is NULL" in detail()
    p = [A + k * base for k in range(12)]
    assert L.gspn_bwd_local(*p, 2, 4, 16, 16, 0xF, 2, -3, 1, 0, A + (40 << 30), 1 << 40, None) == 1
    assert "kchunk" in detail()
    assert L.gspn_bwd_local(*p[:6], None, *p[7:], 2, 4, 16, 16, 0xF, 2, 4, 1, 0, A + (40 << 30), 1 << 40, None) == 1
    assert "dh is NULL" in detail()


def test_merge_validation():
    """gspn_merge_fwd / gspn_merge_bwd (output gate + direction merge, Eq. 2)."""
    L = gspn.lib()
    base = 1 << 30
    h, u, y = A, A + base, A + 2 * base
    assert L.gspn_merge_fwd(None, u, y, 1, 4, 8, 8, 0xF, 1, 0, None) == 1 and "h is NULL" in detail()
    assert L.gspn_merge_fwd(h, u + 2, y, 1, 4, 8, 8, 0xF, 1, 0, None) == 1 and "u is not 16-byte" in detail()
    assert L.gspn_merge_fwd(h, u, y, 1, 4, 8, 8, 0x0, 1, 0, None) == 1 and "dirs" in detail()
    assert L.gspn_merge_fwd(h, u, y, 1, 4, 8, 8, 0xF, 1, 0x1, None) == 1 and "flags" in detail()
    assert L.gspn_merge_fwd(h, u, y, 0, 4, 8, 8, 0xF, 1, 0, None) == 1 and "B must be" in detail()
    assert L.gspn_merge_fwd(h, u, h + 64, 1, 4, 8, 8, 0xF, 1, 0, None) == 1 and "overlaps" in detail()
    dy, dh, du = A + 3 * base, A + 4 * base, A + 5 * base
    assert L.gspn_merge_bwd(h, u, None, dh, du, 1, 4, 8, 8, 0xF, 1, 0, None) == 1 and "dy is NULL" in detail()
    assert L.gspn_merge_bwd(h, u, dy, dh, dh + 16, 1, 4, 8, 8, 0xF, 1, 4, None) == 1 and "overlaps" in detail()
    assert L.gspn_merge_bwd(h, u, dy, u, du, 1, 4, 8, 8, 0xF, 1, 4, None) == 1 and "overlaps" in detail()


def test_proxy_validation():
    """gspn_proxy_mix / gspn_proxy_wgrad (1x1 proxy projections) validate before any CUDA call."""
    L = gspn.lib()
    base = 1 << 30
    i, m, o = A, A + base, A + 2 * base
    assert L.gspn_proxy_mix(None, m, o, 2, 384, 8, 28, 28, 1, 0, None) == 1 and "in is NULL" in detail()
    assert L.gspn_proxy_mix(i, m + 4, o, 2, 384, 8, 28, 28, 1, 0, None) == 1 and "M is not 16-byte" in detail()
    assert L.gspn_proxy_mix(i, m, o, 2, 384, 0, 28, 28, 1, 0, None) == 1 and "Co must be" in detail()
    assert L.gspn_proxy_mix(i, m, o, 2, 384, 8, 28, 28, 1, 0x1, None) == 1 and "flags" in detail()
    assert L.gspn_proxy_mix(i, m, o, 2, 384, 8, 5, 5, 1, 0, None) == 2 and "even" in detail()
    assert L.gspn_proxy_mix(i, m, i + 32, 2, 384, 8, 28, 28, 1, 0, None) == 1 and "overlaps" in detail()
    assert L.gspn_proxy_wgrad(i, m, None, 2, 384, 8, 28, 28, 1, None) == 1 and "dM is NULL" in detail()
    assert L.gspn_proxy_wgrad(i, m, o, 2, 4096, 64, 28, 28, 1, None) == 2


def test_missing_library_fails_loudly(monkeypatch):
    """No CPU fallback: without the built CUDA library the binding raises instead of computing anything."""
    from paper_2512_07884_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIBGSPN", "/nonexistent/libgspn.so")
    with pytest.raises(ImportError, match="not built"):
        _lib.lib()


# ---------------------------------------------------------------- binding shape checks (before any CUDA call)

def _bind_inputs(B=1, C=4, G=4, H=8, W=8, dirs=0xF):
    import torch

    D = bin(dirs).count("1")
    x = torch.zeros(B, C, H, W)
    w = [torch.zeros(D, B, G, H, W) for _ in range(3)]
    lam = torch.zeros(D, B, C, H, W)
    return x, w, lam


@pytest.mark.parametrize("bad", ["w_l", "lam", "h", "dh", "dx", "dw_m", "dlam", "dirs"])
def test_bwd_rejects_mis_shaped_tensors(bad):
    """A mis-shaped tensor must raise ValueError in the binding: the ABI sees only pointers."""
    import torch

    x, (wl, wm, wr), lam = _bind_inputs()
    h, dh = torch.zeros_like(lam), torch.zeros_like(lam)
    outs = [torch.zeros_like(x), torch.zeros_like(wl), torch.zeros_like(wm), torch.zeros_like(wr),
            torch.zeros_like(lam)]
    dirs = 0xF
    if bad == "w_l":
        wl = torch.zeros(4, 1, 2, 8, 8)
    elif bad == "lam":
        lam = torch.zeros(4, 1, 4, 8, 9)
    elif bad == "h":
        h = torch.zeros(3, 1, 4, 8, 8)
    elif bad == "dh":
        dh = torch.zeros(1, 4, 8, 8)  # the merged dy passed as dh
    elif bad == "dx":
        outs[0] = torch.zeros(1, 4, 8, 7)
    elif bad == "dw_m":
        outs[2] = torch.zeros(4, 1, 1, 8, 8)
    elif bad == "dlam":
        outs[4] = torch.zeros(4, 2, 4, 8, 8)
    elif bad == "dirs":
        dirs = 0x3  # D = 2 does not match the 4 direction slabs
    with pytest.raises(ValueError, match="shape"):
        gspn.bwd(x, wl, wm, wr, lam, h, dh, dirs, 4, outs=tuple(outs))


def test_fwd_and_aux_reject_mis_shaped_outputs():
    import torch

    x, (wl, wm, wr), lam = _bind_inputs()
    with pytest.raises(ValueError, match="shape"):
        gspn.fwd(x, wl, wm, wr, lam, 0xF, 4, out=torch.zeros(4, 1, 4, 8, 7))
    h = torch.zeros_like(lam)
    with pytest.raises(ValueError, match="shape"):
        gspn.merge_fwd(h, h, 0xF, out=torch.zeros(1, 4, 8, 9))
    with pytest.raises(ValueError, match="shape"):
        gspn.merge_bwd(h, h, torch.zeros(1, 4, 8, 8), 0xF, outs=(torch.zeros_like(h), torch.zeros(4, 1, 4, 8, 1)))
    with pytest.raises(ValueError, match="shape"):
        gspn.proxy_mix(torch.zeros(2, 6, 4, 4), torch.zeros(3, 6), out=torch.zeros(2, 3, 4, 5))
    with pytest.raises(ValueError, match="shape"):
        gspn.proxy_wgrad(torch.zeros(2, 3, 4, 4), torch.zeros(2, 6, 4, 5))
    with pytest.raises(ValueError, match="shape"):
        gspn.proxy_wgrad(torch.zeros(2, 3, 4, 4), torch.zeros(2, 6, 4, 4), out=torch.zeros(6, 3))


def test_proxy_rejects_32bit_overflowing_extents():
    """The proxy kernels index pixels in 32 bits: H*W >= 2^31 must be refused, not truncated."""
    L = gspn.lib()
    st = L.gspn_proxy_mix(A, A, A + (1 << 40), 1, 1, 1, 46341, 46342, 1, 0, None)
    assert st == 2 and "INT32_MAX" in detail()
    st = L.gspn_proxy_wgrad(A, A + (1 << 40), A + (1 << 41), 1, 1, 1, 46341, 46342, 1, None)
    assert st == 2 and "INT32_MAX" in detail()
