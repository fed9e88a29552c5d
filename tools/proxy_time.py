"""Event-timed tcgen05 proxy projections (gspn_proxy_mix down / up, gspn_proxy_wgrad) on the compact blocks of
BASELINE configs[4] (320 <-> 40, 2048^2) and configs[2] (384 <-> 8, 28^2, B = 64); prints ms and GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_07884_b200 as gspn  # noqa: E402

dev = torch.device("cuda:0")


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for (B, C, Cp, H, W) in [(1, 320, 40, 2048, 2048), (64, 384, 8, 28, 28)]:
    g = torch.Generator(device=dev).manual_seed(1)
    x = (torch.rand((B, C, H, W), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    P = ((torch.rand((Cp, C), generator=g, device=dev) * 2 - 1) / C ** 0.5).to(torch.bfloat16)
    Q = ((torch.rand((C, Cp), generator=g, device=dev) * 2 - 1) / Cp ** 0.5).to(torch.bfloat16)
    xp = gspn.proxy_mix(x, P)
    nbytes = 2 * B * H * W * (C + Cp)
    td = timed(lambda: gspn.proxy_mix(x, P))
    tu = timed(lambda: gspn.proxy_mix(xp, Q))
    tw = timed(lambda: gspn.proxy_wgrad(xp, x))
    print(f"B={B} C={C} Cp={Cp} {H}x{W}: down {td:.4f} ms {nbytes / td / 1e6:.0f} GB/s | up {tu:.4f} ms "
          f"{nbytes / tu / 1e6:.0f} GB/s | wgrad {tw:.4f} ms {nbytes / tw / 1e6:.0f} GB/s")
