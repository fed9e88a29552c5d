"""Config-4 step with the output gate + direction merge (NEXT-1): unfused (gspn_fwd, gspn_merge_fwd,
gspn_merge_bwd, gspn_bwd) vs fused backward (gspn_bwd_merged). Prints per-call times (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_07884_b200 as gspn  # noqa: E402
from synth import seed_for  # noqa: E402
from synth.configs import get_config  # noqa: E402
from synth.device import fill_, make_inputs  # noqa: E402

cfg = get_config("4")
dev = torch.device("cuda:0")
t = make_inputs(cfg, dev, with_dh=False)
u = fill_(torch.empty_like(t["lam"]), seed_for(cfg.cfg_id), "u")
dy = fill_(torch.empty_like(t["x"]), seed_for(cfg.cfg_id), "dy")
G, dirs = cfg.G, cfg.dirs
h = torch.empty_like(t["lam"])
y = torch.empty_like(t["x"])
dh, du = torch.empty_like(h), torch.empty_like(h)
outs = (torch.empty_like(t["x"]), torch.empty_like(t["w_l"]), torch.empty_like(t["w_m"]), torch.empty_like(t["w_r"]),
        torch.empty_like(t["lam"]))
ws = torch.empty(gspn.workspace_bytes(cfg.B, cfg.C, cfg.H, cfg.W, dirs, G, gspn.DTYPE_BF16), dtype=torch.uint8, device=dev)
outs_m = outs + (du,)
wsm = torch.empty(gspn.lib().gspn_bwd_merged_workspace_bytes(cfg.B, cfg.C, cfg.H, cfg.W, dirs, G, gspn.DTYPE_BF16),
                  dtype=torch.uint8, device=dev)
a = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


f = timed(lambda: gspn.fwd(*a, dirs, G, out=h))
mf = timed(lambda: gspn.merge_fwd(h, u, dirs, out=y))
mb = timed(lambda: gspn.merge_bwd(h, u, dy, dirs, outs=(dh, du)))
b = timed(lambda: gspn.bwd(*a, h, dh, dirs, G, outs=outs, workspace=ws))
bm = timed(lambda: gspn.bwd_merged(*a, h, u, dy, dirs, G, outs=outs_m, workspace=wsm))
pb = (gspn.last_path(), gspn.last_launch_count())
fm = timed(lambda: gspn.fwd_merged(*a, u, dirs, G, out=y, h_out=h))
pf = (gspn.last_path(), gspn.last_launch_count())
print(pb, pf)
print(f"fwd {f:.3f} merge_fwd {mf:.3f} merge_bwd {mb:.3f} bwd {b:.3f} | unfused step {f + mf + mb + b:.3f} ms"
      f" | fwd_merged {fm:.3f} bwd_merged {bm:.3f} -> fused step {fm + bm:.3f} ms")
