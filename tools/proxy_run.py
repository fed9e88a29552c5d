"""Config-5 compact block (B=1, C=320 <-> C_proxy=40, 2048 x 2048, bf16) through gspn_proxy_mix / _wgrad:
the workload for ncu captures of the tcgen05 projection kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_07884_b200 as gspn  # noqa: E402

B, C, Cp, H, W = 1, 320, 40, 2048, 2048
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
x = (torch.rand((B, C, H, W), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
P = ((torch.rand((Cp, C), generator=g, device=dev) * 2 - 1) / C ** 0.5).to(torch.bfloat16)
Q = ((torch.rand((C, Cp), generator=g, device=dev) * 2 - 1) / Cp ** 0.5).to(torch.bfloat16)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    xp = gspn.proxy_mix(x, P)
    y = gspn.proxy_mix(xp, Q)
    dP = gspn.proxy_wgrad(xp, x)
torch.cuda.synchronize()
