"""Experiment check: the kHF backward (GSPN_HF, horizontal dw in the recurrence) against the default hybrid
on the same inputs -- per-direction normwise differences; exit 1 if any exceeds the dtype's tolerance.

  GSPN_EXPERIMENTS=1 python tools/hf_cmp.py 1,8,8,16,16,15,f32 2,2,2,512,512,15,bf16   # B,C,G,H,W,dirs,dtype
"""
import os
import sys

os.environ["GSPN_EXPERIMENTS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_07884_b200 as gspn  # noqa: E402
from tests.parity_utils import TOL, host_inputs, small_config, to_torch  # noqa: E402

bad = 0
for arg in sys.argv[1:]:
    B, C, G, H, W, dirs, dt = tuple(int(v) if v.isdigit() else v for v in arg.split(","))
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=700)
    t = {n: to_torch(v[0], dt, "cuda") for n, v in host_inputs(cfg).items()}
    a = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])
    h = gspn.fwd(*a, dirs, G)
    os.environ["GSPN_HF"] = "1"
    g1 = gspn.bwd(*a, h, t["dh"], dirs, G)
    os.environ.pop("GSPN_HF")
    g2 = gspn.bwd(*a, h, t["dh"], dirs, G)
    torch.cuda.synchronize()
    line, worst = [arg], 0.0
    for n, i in (("dx", 0), ("dw_l", 1), ("dw_m", 2), ("dw_r", 3), ("dlam", 4)):
        x, y = g1[i].double(), g2[i].double()
        xs, ys = (x.unsqueeze(0), y.unsqueeze(0)) if i == 0 else (x, y)
        errs = [float((xs[k] - ys[k]).abs().max() / ys[k].abs().max().clamp_min(1e-30)) for k in range(xs.shape[0])]
        worst = max(worst, *errs)
        line.append(n + " " + "/".join(f"{e:.1e}" for e in errs))
    bad += worst > TOL[dt]
    print(" ".join(line), "OK" if worst <= TOL[dt] else "FAIL", flush=True)
sys.exit(1 if bad else 0)
