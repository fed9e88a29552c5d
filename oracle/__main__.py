"""Stand-alone CLI of the fp64 oracle (TEST INFRASTRUCTURE: the product path never runs it).

  python -m oracle --config 1                 # whole BASELINE config 1 (fp32, 16 x 16): fwd + bwd
  python -m oracle --config 4 --units 8       # the first 8 units (b, g) of config 4
  python -m oracle --config 2 --units 4 --save out.npz

Inputs come from synth (the seeded counter-based generator shared with the GPU tests); the outputs'
norms and sums are printed, so a run can be compared with another build or machine line by line, and
--save writes every output (h, dx, dw_l, dw_m, dw_r, dlam) for offline comparison.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def main(argv=None) -> int:
    import oracle
    import synth
    from synth.configs import get_config

    ap = argparse.ArgumentParser(prog="python -m oracle")
    ap.add_argument("--config", default="1")
    ap.add_argument("--units", type=int, default=0, help="first N units (b, g); 0 = all")
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    ap.add_argument("--kchunk", type=int, default=0)
    ap.add_argument("--save", default="")
    a = ap.parse_args(argv)
    cfg = get_config(a.config)
    U = cfg.B * cfg.G
    n = U if a.units <= 0 else min(a.units, U)
    Cg, HW, D = cfg.C // cfg.G, cfg.H * cfg.W, cfg.D
    seed = synth.seed_for(cfg.cfg_id)
    # the first n units as a (B' = n, C' = C/G, G' = 1) problem, regenerated from the unsharded indices
    f = lambda v: synth.as_f64(v, cfg.dtype)  # noqa: E731
    x = f(synth.tensor(seed, "x", (n, Cg, cfg.H, cfg.W), cfg.dtype))
    ws = [f(synth.tensor(seed, nm, (D, n, 1, cfg.H, cfg.W), cfg.dtype, 0, n * HW, U * HW)) for nm in ("w_l", "w_m", "w_r")]
    lam = f(synth.tensor(seed, "lam", (D, n, Cg, cfg.H, cfg.W), cfg.dtype, 0, n * Cg * HW, cfg.B * cfg.C * HW))
    dh = f(synth.tensor(seed, "dh", (D, n, Cg, cfg.H, cfg.W), cfg.dtype, 0, n * Cg * HW, cfg.B * cfg.C * HW))
    t0 = time.perf_counter()
    h = oracle.fwd(x, *ws, lam, cfg.dirs, 1, threads=a.threads, kchunk=a.kchunk)
    t1 = time.perf_counter()
    g = oracle.bwd(x, *ws, lam, h, dh, cfg.dirs, 1, threads=a.threads, kchunk=a.kchunk)
    t2 = time.perf_counter()
    outs = {"h": h, "dx": g[0], "dw_l": g[1], "dw_m": g[2], "dw_r": g[3], "dlam": g[4]}
    print(f"config {cfg.name}: {n} of {U} units (b, g), C/G = {Cg}, {cfg.H} x {cfg.W}, dirs {cfg.dirs:#x}, "
          f"{cfg.dtype} inputs, fp64 oracle, {a.threads} threads")
    print(f"fwd {t1 - t0:.3f} s   bwd {t2 - t1:.3f} s")
    for k, v in outs.items():
        print(f"  {k:5s} shape {tuple(v.shape)}  max|.| {np.abs(v).max():.6e}  sum {v.sum():+.9e}")
    if a.save:
        np.savez(a.save, **outs)
        print(f"saved {a.save}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
