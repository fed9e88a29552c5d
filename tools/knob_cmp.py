"""Bitwise comparison of the forward (h) and backward outputs with and without an experiment knob that must not
change results (e.g. GSPN_HCP: horizontal tap tiles by cp.async). Exit 1 on any difference.
  python tools/knob_cmp.py KNOB B,C,G,H,W,dirs,dtype ..."""
import os
import sys

os.environ["GSPN_EXPERIMENTS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_07884_b200 as gspn  # noqa: E402
from tests.parity_utils import host_inputs, small_config, to_torch  # noqa: E402

knob, bad = sys.argv[1], 0
for arg in sys.argv[2:]:
    B, C, G, H, W, dirs, dt = tuple(int(v) if v.isdigit() else v for v in arg.split(","))
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=720)
    t = {n: to_torch(v[0], dt, "cuda") for n, v in host_inputs(cfg).items()}
    a = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])
    outs = []
    for on in (False, True):
        if on:
            os.environ[knob] = "1"
        h = gspn.fwd(*a, dirs, G)
        outs.append((h, *gspn.bwd(*a, h, t["dh"], dirs, G)))
        os.environ.pop(knob, None)
    torch.cuda.synchronize()
    same = [bool(torch.equal(u, v)) for u, v in zip(*outs)]
    bad += not all(same)
    print(arg, knob, "h,dx,dw_l,dw_m,dw_r,dlam bitwise:", same, flush=True)
sys.exit(1 if bad else 0)
