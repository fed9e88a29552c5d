"""Multi-GPU sharding on one GPU: each rank's shard (synth.device.shard_for) is run through
the CUDA path on its own, exactly as bench.py's ranks run it, and compared with the unsharded run.

* unit shards (b, g) -- configs 2/3/4 at N > 1: every output of a unit is unit-local, so the shards'
  h, dlam, dx and dw are bitwise the unsharded ones (same kernels, same per-position arithmetic);
* channel split of a single unit -- config 5 at N > 1: h, dlam, dx are channel-local (bitwise); dw is a
  sum over channels, so each shard emits fp32 partial sums (GSPN_FLAG_DW_F32) whose sum over ranks (what
  the NCCL all-reduce computes) matches the unsharded dw within the north_star tolerance.
"""
from __future__ import annotations

import pytest

import paper_2512_07884_b200 as gspn
from synth.configs import Config
from synth.device import full_shard, make_inputs, shard_for
from tests.parity_utils import TOL, check, from_torch

pytestmark = pytest.mark.gpu


def _run(cfg, sh, dev, flags=0):
    t = make_inputs(cfg, dev, sh)
    h = gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], cfg.dirs, sh.G)
    g = gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], cfg.dirs, sh.G, flags=flags)
    return h, g


UNIT_CASES = [
    Config("u4", 4, 3, 6, 6, 64, 64, 0xF, "bf16", "config-4-like, per-channel"),
    Config("u3b", 3, 2, 12, 3, 28, 28, 0xF, "bf16", "config-3b-like, grouped small planes"),
    Config("u2", 2, 2, 4, 4, 300, 264, 0xF, "f32", "per-channel, unpacked fused path"),
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg", UNIT_CASES, ids=lambda c: c.name)
def test_unit_shards_bitwise(cfg, world, cuda_device):
    import torch

    h0, g0 = _run(cfg, full_shard(cfg), cuda_device)
    Cg = cfg.C // cfg.G
    for rank in range(world):
        sh = shard_for(cfg, rank, world)
        assert sh.kind == "units"
        h, (dx, dwl, dwm, dwr, dlam) = _run(cfg, sh, cuda_device)
        for ub in range(sh.B):
            b, gr = divmod(sh.unit0 + ub, cfg.G)
            cs = slice(gr * Cg, (gr + 1) * Cg)
            assert torch.equal(h[:, ub], h0[:, b, cs]), f"rank {rank} unit {ub}: h"
            assert torch.equal(dlam[:, ub], g0[4][:, b, cs]), f"rank {rank} unit {ub}: dlam"
            assert torch.equal(dx[ub], g0[0][b, cs]), f"rank {rank} unit {ub}: dx"
            for name, a, r in (("dw_l", dwl, g0[1]), ("dw_m", dwm, g0[2]), ("dw_r", dwr, g0[3])):
                assert torch.equal(a[:, ub, 0], r[:, b, gr]), f"rank {rank} unit {ub}: {name}"


CHANNEL_CASES = [
    Config("c5", 5, 1, 8, 1, 96, 128, 0xF, "bf16", "config-5-like: one unit, shared w"),
    Config("c5f", 5, 1, 8, 1, 40, 600, 0xF, "f32", "one unit, P-split chains"),  # >= 2 channels per rank
]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cfg", CHANNEL_CASES, ids=lambda c: c.name)
def test_channel_split_partial_dw(cfg, world, cuda_device):
    import torch

    h0, g0 = _run(cfg, full_shard(cfg), cuda_device)
    dw_sum = [torch.zeros(g0[1].shape, dtype=torch.float64, device=cuda_device) for _ in range(3)]
    for rank in range(world):
        sh = shard_for(cfg, rank, world)
        assert sh.kind == "channels"
        h, (dx, dwl, dwm, dwr, dlam) = _run(cfg, sh, cuda_device, flags=gspn.FLAG_DW_F32)
        assert dwl.dtype == torch.float32
        cs = slice(sh.chan0, sh.chan0 + sh.chans)
        assert torch.equal(h, h0[:, :, cs]), f"rank {rank}: h"
        assert torch.equal(dlam, g0[4][:, :, cs]), f"rank {rank}: dlam"
        assert torch.equal(dx, g0[0][:, cs]), f"rank {rank}: dx"
        for i, a in enumerate((dwl, dwm, dwr)):
            dw_sum[i] += a.to(torch.float64)
    for i, n in enumerate(("dw_l", "dw_m", "dw_r")):
        check(f"channel_split[{cfg.name},{world}]", n, from_torch(dw_sum[i]), from_torch(g0[1 + i]), TOL[cfg.dtype])


def test_dw_f32_flag_matches_io_dtype_dw(cuda_device):
    """GSPN_FLAG_DW_F32 changes only the dw storage: rounding its fp32 output to bf16 gives the bf16 dw."""
    import torch

    cfg = Config("f", 5, 2, 8, 2, 40, 56, 0xF, "bf16", "grouped")
    sh = full_shard(cfg)
    _, g = _run(cfg, sh, cuda_device)
    _, g32 = _run(cfg, sh, cuda_device, flags=gspn.FLAG_DW_F32)
    for i in (1, 2, 3):
        assert g32[i].dtype == torch.float32
        assert torch.equal(g32[i].to(torch.bfloat16), g[i])
    for i in (0, 4):
        assert torch.equal(g32[i], g[i])
