"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host logic: unit sharding with no
data-path collective, and the single-unit channel split whose partial dw are all-reduced.

Each rank regenerates exactly its shard of the inputs from the unsharded flat indices, runs the
oracle on it, and the gathered shard results must equal the unsharded run (bitwise for the per-unit
quantities; within fp64 rounding for the all-reduced dw).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_on(cfg, inp, G):
    import oracle
    import synth

    f = {k: synth.as_f64(v, cfg.dtype) for k, v in inp.items()}
    h = oracle.fwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], cfg.dirs, G)
    g = oracle.bwd(f["x"], f["w_l"], f["w_m"], f["w_r"], f["lam"], h, f["dh"], cfg.dirs, G)
    return h, g


def _worker(rank, world, port, cfg_kw, outdir):
    import sys

    sys.path.insert(0, ROOT)
    from synth.configs import get_config
    from synth.device import host_shard_inputs, shard_for

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = get_config(cfg_kw.pop("base")).with_(**cfg_kw)
    sh = shard_for(cfg, rank, world)
    inp = host_shard_inputs(cfg, sh)
    h, (dx, dwl, dwm, dwr, dlam) = _oracle_on(cfg, inp, sh.G)
    if sh.kind == "channels":
        # the only exchange of the path: partial dw (linear in the channels' contributions) summed
        for a in (dwl, dwm, dwr):
            t = torch.from_numpy(a)
            dist.all_reduce(t)
            a[...] = t.numpy()
    # gather everything to rank 0 (test plumbing, not part of the data path)
    payload = {"h": h, "dx": dx, "dlam": dlam, "dwl": dwl, "dwm": dwm, "dwr": dwr, "kind": sh.kind}
    objs = [None] * world
    dist.all_gather_object(objs, payload)
    if rank == 0:
        np.save(os.path.join(outdir, "gathered.npy"), np.array(objs, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def _run(cfg_kw, tmp_path):
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, dict(cfg_kw), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    return list(np.load(os.path.join(tmp_path, "gathered.npy"), allow_pickle=True))


def test_unit_sharding_equals_unsharded(tmp_path):
    from synth.configs import get_config
    from synth.device import host_shard_inputs

    kw = dict(base="2", B=3, C=4, G=2, H=6, W=5)
    parts = _run(kw, tmp_path)
    cfg = get_config("2").with_(**{k: v for k, v in kw.items() if k != "base"})
    h, (dx, dwl, dwm, dwr, dlam) = _oracle_on(cfg, host_shard_inputs(cfg), cfg.G)
    D, B, C, G, H, W = cfg.D, cfg.B, cfg.C, cfg.G, cfg.H, cfg.W
    Cg = C // G
    assert all(p["kind"] == "units" for p in parts)
    # units are (b, g) flattened; a shard's local [D, U', Cg, H, W] concatenates along units
    cat = lambda key: np.concatenate([p[key].reshape(D, -1) for p in parts], axis=1)
    np.testing.assert_array_equal(cat("h"), h.reshape(D, -1))
    np.testing.assert_array_equal(cat("dlam"), dlam.reshape(D, -1))
    np.testing.assert_array_equal(np.concatenate([p["dx"].reshape(-1) for p in parts]), dx.reshape(-1))
    for key, ref in (("dwl", dwl), ("dwm", dwm), ("dwr", dwr)):
        np.testing.assert_array_equal(cat(key), ref.reshape(D, -1))


def test_channel_split_allreduce_equals_unsharded(tmp_path):
    from synth.configs import get_config
    from synth.device import host_shard_inputs

    kw = dict(base="5", B=1, C=6, G=1, H=8, W=6)
    parts = _run(kw, tmp_path)
    cfg = get_config("5").with_(**{k: v for k, v in kw.items() if k != "base"})
    h, (dx, dwl, dwm, dwr, dlam) = _oracle_on(cfg, host_shard_inputs(cfg), 1)
    D = cfg.D
    assert all(p["kind"] == "channels" for p in parts)
    np.testing.assert_array_equal(np.concatenate([p["h"] for p in parts], axis=2), h)
    np.testing.assert_array_equal(np.concatenate([p["dlam"] for p in parts], axis=2), dlam)
    np.testing.assert_array_equal(np.concatenate([p["dx"] for p in parts], axis=1), dx)
    for key, ref in (("dwl", dwl), ("dwm", dwm), ("dwr", dwr)):
        for p in parts:
            np.testing.assert_allclose(p[key], ref, rtol=0, atol=1e-13 * max(1.0, np.abs(ref).max()))


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-executes itself under torch.distributed.run (2 ranks, rendezvous on
    127.0.0.1). Exercised through the CPU-only reference arm: rank 0 alone prints one JSON line, rank 1 exits 0."""
    import json
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                          "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0", "--config", "1", "--cpu-seconds", "0.2"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2
