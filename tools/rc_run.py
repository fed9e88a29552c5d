"""Config 4 through gspn_fwd_ckpt + gspn_bwd_recompute (NEXT-3): the workload for an ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_07884_b200 as gspn  # noqa: E402
from synth.configs import get_config  # noqa: E402
from synth.device import make_inputs  # noqa: E402

cfg = get_config("4")
dev = torch.device("cuda:0")
t = make_inputs(cfg, dev)
a = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])
for _ in range(2):
    ck, _ = gspn.fwd_ckpt(*a, cfg.dirs, cfg.G)
    gspn.bwd_recompute(*a, ck, t["dh"], cfg.dirs, cfg.G)
torch.cuda.synchronize()
