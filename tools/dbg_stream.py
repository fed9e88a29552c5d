"""Debug helper: one small fwd/bwd through the stream path, synchronising after each call."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_07884_b200 as gspn
from tests.parity_utils import small_config, host_inputs, to_torch
shape = tuple(int(v) for v in sys.argv[1:7]) if len(sys.argv) > 6 else (1, 8, 8, 16, 16, 4)
dtype = sys.argv[7] if len(sys.argv) > 7 else "f32"
B, C, G, H, W, dirs = shape
cfg = small_config(B, C, G, H, W, dirs, dtype)
inp = host_inputs(cfg)
dev = torch.device("cuda:0")
t = {k: to_torch(v[0], dtype, dev) for k, v in inp.items()}
h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], dirs, G)
print("fwd path", gspn.last_path(), flush=True)
torch.cuda.synchronize()
print("fwd ok", flush=True)
g = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], dirs, G)
print("bwd path", gspn.last_path(), flush=True)
torch.cuda.synchronize()
print("bwd ok", flush=True)
