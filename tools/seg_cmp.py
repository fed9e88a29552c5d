"""GSPN-local segment work items (NEXT-2 as a scheduler) against the same kchunk on the global schedule
(experiment knob GSPN_NO_SEGITEMS): h, dx, dw, dlam must be BITWISE equal -- a segment starts from h = 0 and
g = 0 either way, only the order of work items changes. Exit 1 on any difference.

  python tools/seg_cmp.py 1,8,8,512,512,15,bf16,128 ...     # B,C,G,H,W,dirs,dtype,kchunk
"""
import os
import sys

os.environ["GSPN_EXPERIMENTS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_07884_b200 as gspn  # noqa: E402
from tests.parity_utils import host_inputs, small_config, to_torch  # noqa: E402

bad = 0
for arg in sys.argv[1:]:
    B, C, G, H, W, dirs, dt, k = tuple(int(v) if v.isdigit() else v for v in arg.split(","))
    cfg = small_config(B, C, G, H, W, dirs, dt, cfg_id=710)
    t = {n: to_torch(v[0], dt, "cuda") for n, v in host_inputs(cfg).items()}
    a = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])
    outs = []
    for off in (False, True):
        if off:
            os.environ["GSPN_NO_SEGITEMS"] = "1"
        h = gspn.fwd(*a, dirs, G, kchunk=k)
        g = gspn.bwd(*a, h, t["dh"], dirs, G, kchunk=k)
        outs.append((h, *g))
        os.environ.pop("GSPN_NO_SEGITEMS", None)
    torch.cuda.synchronize()
    same = [bool(torch.equal(u, v)) for u, v in zip(*outs)]
    ok = all(same)
    bad += not ok
    print(arg, "h,dx,dw_l,dw_m,dw_r,dlam bitwise:", same, "OK" if ok else "FAIL", flush=True)
sys.exit(1 if bad else 0)
