"""Event-timed GSPN-local (kchunk) fwd + bwd against the global scan on one shape; with
GSPN_EXPERIMENTS=1 GSPN_NO_SEGITEMS=1 the segments run on the global schedule (kchunk as a model variant
only). Prints one line: shape, kchunk, fwd / bwd ms, and a checksum of h (bitwise comparison across runs).
  python tools/local_time.py B C G H W kchunk"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_07884_b200 as gspn  # noqa: E402

B, C, G, H, W, k = (int(v) for v in sys.argv[1:7])
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(3)
bf = torch.bfloat16
x = (torch.rand((B, C, H, W), generator=g, device=dev) * 2 - 1).to(bf)
w = [(torch.rand((4, B, G, H, W), generator=g, device=dev) * 0.95 + 0.05).to(bf) for _ in range(3)]
lam = torch.rand((4, B, C, H, W), generator=g, device=dev).to(bf)
dh = (torch.rand((4, B, C, H, W), generator=g, device=dev) * 2 - 1).to(bf)


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for kc in ([0, k] if k else [0]):
    h = gspn.fwd(x, *w, lam, 0xF, G, kchunk=kc)
    tf = timed(lambda: gspn.fwd(x, *w, lam, 0xF, G, kchunk=kc))
    tb = timed(lambda: gspn.bwd(x, *w, lam, h, dh, 0xF, G, kchunk=kc))
    grads = gspn.bwd(x, *w, lam, h, dh, 0xF, G, kchunk=kc)
    torch.cuda.synchronize()
    cs = float(h.float().abs().sum()) + sum(float(t.float().abs().sum()) for t in grads)
    print(f"B={B} C={C} G={G} {H}x{W} kchunk={kc}: fwd {tf:.4f} ms bwd {tb:.4f} ms path {gspn.last_path()} "
          f"checksum {cs:.9e}", flush=True)
