#!/usr/bin/env python
"""Benchmark of the GSPN line-scan hot path (fwd + bwd, all directions) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One "step" = one gspn_fwd + one gspn_bwd call (every SURVEY.md §8(a) row) over one batch of synthetic,
device-generated inputs already resident in HBM. Metric (BASELINE.json): algorithmic HBM GB/s of the
fwd+bwd scan, (bytes_fwd + bytes_bwd) / device time, bytes per SURVEY.md §8(d). Multi-GPU: one process
per GPU (torchrun), units (b, g) sharded across ranks with no data-path collective; by default each
rank owns one full configuration's worth of units (weak scaling); --scaling strong splits the one
configuration instead (config 5 then needs the dw all-reduce over NCCL). Timing: CUDA events on the
launching stream, barrier + synchronize around the timed region, max over ranks.

--impl reference times the fp64 CPU oracle (oracle/, the tier's reference arm) on bounded samples of
the same workload on this host's cores; it never touches the GPU path.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GSPN fwd+bwd scan GB/s vs B200 HBM peak; latency @1/2/4/8 GPUs"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the SURVEY §8(f) rows (merge, GSPN-local)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--dirs", type=lambda v: int(v, 0), default=None, help="override the direction mask (experiments)")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                maxs.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def traffic_for(config_name: str, kernel: str):
    try:
        with open(TRAFFIC_FILE) as f:
            t = json.load(f)
        return t.get(config_name, {}).get(kernel)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------ oracle arm

def oracle_prepare(cfg, max_elems: int = 1 << 27):
    """A bounded sample of `cfg` for the CPU oracle: consecutive units (b, g) as one (B'=n, C=C/G, G=1)
    problem whose largest tensor has at most `max_elems` elements, inputs regenerated on the host (fp64).
    Generated once (untimed); `oracle_time` then times passes over it."""
    import oracle
    import synth

    U = cfg.B * cfg.G
    Cg = cfg.C // cfg.G
    HW = cfg.H * cfg.W
    D = cfg.D
    n_units = int(max(1, min(U, max_elems // max(1, D * Cg * HW))))
    seed = synth.seed_for(cfg.cfg_id)
    x = synth.as_f64(synth.tensor(seed, "x", (n_units, Cg, cfg.H, cfg.W), cfg.dtype), cfg.dtype)
    ws = [synth.as_f64(synth.tensor(seed, n, (D, n_units, 1, cfg.H, cfg.W), cfg.dtype, 0, n_units * HW,
                                    U * HW), cfg.dtype) for n in ("w_l", "w_m", "w_r")]
    lam = synth.as_f64(synth.tensor(seed, "lam", (D, n_units, Cg, cfg.H, cfg.W), cfg.dtype, 0,
                                    n_units * Cg * HW, cfg.B * cfg.C * HW), cfg.dtype)
    dh = synth.as_f64(synth.tensor(seed, "dh", (D, n_units, Cg, cfg.H, cfg.W), cfg.dtype, 0,
                                   n_units * Cg * HW, cfg.B * cfg.C * HW), cfg.dtype)
    unit_cfg = cfg.with_(B=1, C=Cg, G=1)
    per_unit = unit_cfg.fwd_bytes() + unit_cfg.bwd_bytes()
    threads = oracle.default_threads()
    desc = (f"{n_units} of {U} units (b,g) of config {cfg.name} (fwd+bwd, all {D} directions, fp64 oracle, "
            f"{threads} threads); bytes counted at the I/O dtype")
    return {"x": x, "ws": ws, "lam": lam, "dh": dh, "dirs": cfg.dirs, "bytes": n_units * per_unit,
            "threads": threads, "desc": desc}


def oracle_time(sm, seconds: float):
    """Time whole fwd+bwd passes of the oracle (as it stands) over a prepared sample until ~`seconds`
    (at least one pass). Returns (algorithmic bytes processed, wall seconds, threads, description)."""
    import oracle

    passes, t0 = 0, time.perf_counter()
    while True:
        h = oracle.fwd(sm["x"], *sm["ws"], sm["lam"], sm["dirs"], 1, threads=sm["threads"])
        oracle.bwd(sm["x"], *sm["ws"], sm["lam"], h, sm["dh"], sm["dirs"], 1, threads=sm["threads"])
        passes += 1
        wall = time.perf_counter() - t0
        if wall >= seconds:
            break
    return passes * sm["bytes"], wall, sm["threads"], f"{sm['desc']}; {passes} pass(es)"


def oracle_sample(cfg, seconds: float):
    return oracle_time(oracle_prepare(cfg), seconds)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from synth.configs import get_config

    cfg = get_config(args.config)
    per_step = max(2.0, min(args.cpu_seconds, 60.0 / max(1, args.steps + args.warmup)))
    sm = oracle_prepare(cfg)
    for _ in range(args.warmup):
        oracle_time(sm, per_step / 2)
    vals, walls, desc, threads = [], [], "", 1
    for _ in range(args.steps):
        b, w, threads, desc = oracle_time(sm, per_step)
        vals.append(b / w / 1e9)
        walls.append(w)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(walls) * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based generator)",
        "config": {"workload": f"config {cfg.name}: {cfg.text}", "sample": desc},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2512_07884_b200 as gspn
    from synth.configs import get_config
    from synth.device import make_inputs, shard_for

    rank, world, local = dist_env()
    if world != args.gpus:
        if rank == 0:
            print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    base = get_config(args.config)
    if args.dirs is not None:
        base = base.with_(dirs=args.dirs)
    if args.scaling == "weak":
        gcfg = base.with_(B=base.B * world)  # each rank owns one configuration's worth of units
    else:
        gcfg = base
    sh = shard_for(gcfg, rank, world)
    t = make_inputs(gcfg, dev, sh)
    D = gcfg.D
    dt_code = gspn.DTYPE_BF16 if gcfg.dtype == "bf16" else gspn.DTYPE_F32
    h = torch.empty_like(t["lam"])
    outs = (torch.empty_like(t["x"]), torch.empty_like(t["w_l"]), torch.empty_like(t["w_m"]),
            torch.empty_like(t["w_r"]), torch.empty_like(t["lam"]))
    wsb = gspn.workspace_bytes(sh.B, sh.C, gcfg.H, gcfg.W, gcfg.dirs, sh.G, dt_code)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    bytes_f = gspn.algorithmic_bytes(sh.B, sh.C, gcfg.H, gcfg.W, gcfg.dirs, sh.G, dt_code, False)
    bytes_b = gspn.algorithmic_bytes(sh.B, sh.C, gcfg.H, gcfg.W, gcfg.dirs, sh.G, dt_code, True)
    need_allreduce = sh.kind == "channels"  # one unit split by channel: dw partial sums must be reduced
    work_bytes = sum(v.numel() * v.element_size() for v in t.values() if v is not None) + \
        h.numel() * h.element_size() + sum(o.numel() * o.element_size() for o in outs)
    flush = work_bytes < 4 * L2_BYTES
    flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev) if flush else None
    stream = torch.cuda.current_stream(dev)
    launches = {"fwd": 0, "bwd": 0}

    def step(evs=None):
        if evs:
            evs[0].record(stream)
        gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], gcfg.dirs, sh.G, flags=args.flags, out=h)
        launches["fwd"] = gspn.last_launch_count()
        if evs:
            evs[1].record(stream)
        gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], gcfg.dirs, sh.G, flags=args.flags,
                 outs=outs, workspace=ws)
        launches["bwd"] = gspn.last_launch_count()
        if need_allreduce:
            for o in outs[1:4]:
                dist.all_reduce(o)  # bf16/fp32 in place; NCCL over NVLink
        if evs:
            evs[2].record(stream)

    for _ in range(args.warmup):
        step()
        if flush:
            flush_buf.zero_()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    evs_all = []
    t_wall0 = time.perf_counter()
    ev_start = torch.cuda.Event(enable_timing=True)
    ev_end = torch.cuda.Event(enable_timing=True)
    ev_start.record(stream)
    for _ in range(args.steps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        step(evs)
        evs_all.append(evs)
        if flush:
            flush_buf.zero_()
    ev_end.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    f_ms = [e[0].elapsed_time(e[1]) for e in evs_all]
    b_ms = [e[1].elapsed_time(e[2]) for e in evs_all]
    step_ms = sum(f_ms[i] + b_ms[i] for i in range(args.steps)) / args.steps
    region_ms = ev_start.elapsed_time(ev_end) / args.steps
    mean_f, mean_b = sum(f_ms) / len(f_ms), sum(b_ms) / len(b_ms)
    stats = torch.tensor([step_ms, mean_f, mean_b], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    step_ms, mean_f, mean_b = [float(v) for v in stats.tolist()]
    total_bytes = (bytes_f + bytes_b) * world  # every rank processes the same amount of work
    if args.scaling == "strong":
        total_bytes = gcfg.fwd_bytes() + gcfg.bwd_bytes()

    # ---- SURVEY §8(f) rows on the same workload (after the headline region; not part of `value`)
    nxt = None
    if not args.no_next:
        nxt = measure_next(args, gspn, gcfg, sh, t, h, outs, ws, dev, stream)

    # ---- end to end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, gspn, gcfg, sh, t, h, outs, ws, dev, world, dist)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            b_cpu, w_cpu, thr, desc = oracle_sample(base, args.cpu_seconds)
            cpu = {"value": b_cpu / w_cpu / 1e9, "unit": "GB/s", "cores": thr, "kind": "oracle", "sample": desc}
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0
    peak, peak_src = peaks()
    dominant = "bwd" if bytes_b / max(mean_b, 1e-9) <= bytes_f / max(mean_f, 1e-9) or mean_b >= mean_f else "fwd"
    dom_ms = mean_b if dominant == "bwd" else mean_f
    dom_bytes = bytes_b if dominant == "bwd" else bytes_f
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    value = total_bytes / (step_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": gcfg.dtype,
        "data": "synthetic (seeded counter-based generator, device-generated; SURVEY.md §8(d) distributions)",
        "config": {
            "workload": f"config {base.name} (BASELINE.json configs[{base.cfg_id - 1}]): {base.text}",
            "B": gcfg.B, "C": gcfg.C, "G": gcfg.G, "H": gcfg.H, "W": gcfg.W, "dirs": gcfg.dirs,
            "per_rank": {"B": sh.B, "C": sh.C, "G": sh.G, "kind": sh.kind},
            "fwd_ms": mean_f, "bwd_ms": mean_b, "region_ms_per_step": region_ms,
            "fwd_gbs": bytes_f / (mean_f * 1e-3) / 1e9, "bwd_gbs": bytes_b / (mean_b * 1e-3) / 1e9,
            "algorithmic_bytes_per_step": total_bytes,
            "l2": ("L2 flushed (2x126 MB memset) between steps, outside the event pairs" if flush else
                   f"inputs+outputs {work_bytes / 1e9:.1f} GB > 126 MB L2, no flush"),
            "path": gspn.last_path(),
            "wall_s_timed_region": t_wall,
        },
        "roofline": {
            "bound": "hbm", "kernel": f"gspn_{dominant} ({gspn.last_path()} path)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": peak_src,
            "traffic": traffic_for(base.name, dominant),
            "algorithmic_bytes_per_launch": dom_bytes,
        },
        "clocks": clk,
        "gpu_launches": args.steps * (launches["fwd"] + launches["bwd"]),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "next": nxt,
    }
    print(json.dumps(line), flush=True)
    return 0


def measure_next(args, gspn, cfg, sh, t, h, outs, ws, dev, stream):
    """SURVEY §8(f) rows on the bench workload, each timed alone with CUDA events after warm-up:
    NEXT-1 output gate + direction merge (gspn_merge_fwd / _bwd; algorithmic bytes s N (2D+1) and
    s N (4D+1), one launch each) and NEXT-2 GSPN-local fwd + bwd (kchunk = L/4; same bytes as the
    global scan)."""
    import torch

    from synth import seed_for
    from synth.device import fill_

    peak, _ = peaks()
    D, s = cfg.D, (2 if cfg.dtype == "bf16" else 4)
    N = sh.B * sh.C * cfg.H * cfg.W
    seed = seed_for(cfg.cfg_id)
    u = fill_(torch.empty_like(h), seed, "u")
    dy = fill_(torch.empty_like(t["x"]), seed, "dy")
    y = torch.empty_like(t["x"])
    dh2, du = torch.empty_like(h), torch.empty_like(h)

    def timed(fn, reps):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps

    reps = max(3, args.steps)
    out = {}
    mf = timed(lambda: gspn.merge_fwd(h, u, cfg.dirs, out=y), reps)
    mb = timed(lambda: gspn.merge_bwd(h, u, dy, cfg.dirs, outs=(dh2, du)), reps)
    for name, ms, nbytes in (("merge_fwd", mf, s * N * (2 * D + 1)), ("merge_bwd", mb, s * N * (4 * D + 1))):
        gbs = nbytes / (ms * 1e-3) / 1e9
        out[name] = {"ms": ms, "gbs": gbs, "frac": gbs / peak, "bytes": nbytes, "launches": 1}
    del u, dy, y, dh2, du
    k = max(1, min(cfg.H, cfg.W) // 4)
    lf = timed(lambda: gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], cfg.dirs, sh.G, out=h, kchunk=k), reps)
    lpath = gspn.last_path()
    lb = timed(lambda: gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], h, t["dh"], cfg.dirs, sh.G,
                                outs=outs, workspace=ws, kchunk=k), reps)
    bf = gspn.algorithmic_bytes(sh.B, sh.C, cfg.H, cfg.W, cfg.dirs, sh.G,
                                gspn.DTYPE_BF16 if cfg.dtype == "bf16" else gspn.DTYPE_F32, False)
    out["local"] = {"kchunk": k, "fwd_ms": lf, "bwd_ms": lb, "gbs": 3 * bf / ((lf + lb) * 1e-3) / 1e9,
                    "path": lpath}
    out["local"]["frac"] = out["local"]["gbs"] / peak
    # NEXT-4: proxy projections on BASELINE configs[2]'s compact block (B=64, C=384 -> C_proxy=8, 28 x 28)
    pB, pC, pCp, pH, pW = 64, 384, 8, 28, 28
    dtp = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(7884)
    xin = (torch.rand((pB, pC, pH, pW), generator=g, device=dev) * 2 - 1).to(dtp)
    Pd = ((torch.rand((pCp, pC), generator=g, device=dev) * 2 - 1) / pC ** 0.5).to(dtp)
    Qu = ((torch.rand((pC, pCp), generator=g, device=dev) * 2 - 1) / pCp ** 0.5).to(dtp)
    xp = torch.empty((pB, pCp, pH, pW), dtype=dtp, device=dev)
    yo = torch.empty_like(xin)
    dPd = torch.empty((pCp, pC), dtype=torch.float32, device=dev)
    md = timed(lambda: gspn.proxy_mix(xin, Pd, out=xp), reps)
    mu = timed(lambda: gspn.proxy_mix(xp, Qu, out=yo), reps)
    mw = timed(lambda: gspn.proxy_wgrad(xp, xin, out=dPd), reps)
    nb = 2 * pB * pH * pW * (pC + pCp)
    out["proxy"] = {"shape": f"B={pB} C={pC} C_proxy={pCp} {pH}x{pW} bf16",
                    "down_ms": md, "down_gbs": nb / (md * 1e-3) / 1e9, "up_ms": mu, "up_gbs": nb / (mu * 1e-3) / 1e9,
                    "wgrad_ms": mw, "wgrad_gbs": nb / (mw * 1e-3) / 1e9, "bytes": nb}
    return out


def run_e2e(args, gspn, cfg, sh, t, h, outs, ws, dev, world, dist):
    """Same metric through the public API with pinned HOST buffers: every step copies all of its inputs
    host->device, runs fwd + bwd, and copies every output device->host, inside the CUDA-event timed
    region. The batch is streamed in (b, group-block) chunks (units are independent) through two
    device buffer sets on three streams, so H2D of chunk k+1, compute of chunk k and D2H of chunk k-1
    overlap (PCIe is full duplex) -- the way a caller with host-resident data uses the API."""
    import torch

    names = ["x", "w_l", "w_m", "w_r", "lam", "dh"]
    onames = ["h", "dx", "dw_l", "dw_m", "dw_r", "dlam"]
    host_in = {}
    for n in names:
        host_in[n] = torch.empty(t[n].shape, dtype=t[n].dtype, pin_memory=True)
        host_in[n].copy_(t[n])
    full_out = {"h": h, "dx": outs[0], "dw_l": outs[1], "dw_m": outs[2], "dw_r": outs[3], "dlam": outs[4]}
    host_out = {n: torch.empty(full_out[n].shape, dtype=full_out[n].dtype, pin_memory=True) for n in onames}
    h2d = sum(v.numel() * v.element_size() for v in host_in.values())
    d2h = sum(v.numel() * v.element_size() for v in host_out.values())
    B, G = sh.B, sh.G
    Cg = sh.C // sh.G
    dt_code = gspn.DTYPE_BF16 if cfg.dtype == "bf16" else gspn.DTYPE_F32
    wnames = {"w_l", "w_m", "w_r", "dw_l", "dw_m", "dw_r"}
    # ~16 chunks of consecutive units per step, so the pipeline fill / drain is short:
    #  G > 1: (one b, a block of gb groups);  G = 1 (unit shards, compact configs): a block of cb batches
    if G > 1:
        nsub = max(1, 16 // max(1, B))
        while G % nsub:
            nsub -= 1
        gb, cb = G // nsub, 1
        chunks = [(b, 1, k * gb) for b in range(B) for k in range(nsub)]
    else:
        gb, cb = 1, max(1, -(-B // 16))
        while B % cb:  # equal chunks: every chunk buffer view stays contiguous
            cb += 1
        chunks = [(b, cb, 0) for b in range(0, B, cb)]

    def piece(x, b, nb, g0, is_w):  # contiguous pieces of chunk (batches b..b+nb, groups g0..g0+gb)
        lo, hi = (g0, g0 + gb) if is_w else (g0 * Cg, (g0 + gb) * Cg)
        if nb > 1:  # G = 1: whole batches
            return [x[b:b + nb]] if x.dim() == 4 else [x[d, b:b + nb] for d in range(x.shape[0])]
        return [x[b, lo:hi]] if x.dim() == 4 else [x[d, b, lo:hi] for d in range(x.shape[0])]

    def dshape(x, is_w):
        n = gb if is_w else gb * Cg
        return (cb, n) + tuple(x.shape[2:]) if x.dim() == 4 else (x.shape[0], cb, n) + tuple(x.shape[3:])

    def view(x, nb):  # the first nb batches of a chunk buffer (a short last chunk)
        return x[:nb] if x.dim() == 4 else x[:, :nb]

    bufs = []
    for _ in range(2):
        bi = {n: torch.empty(dshape(t[n], n in wnames), dtype=t[n].dtype, device=dev) for n in names}
        bo = {n: torch.empty(dshape(full_out[n], n in wnames), dtype=full_out[n].dtype, device=dev) for n in onames}
        wsb = gspn.workspace_bytes(cb, gb * Cg, cfg.H, cfg.W, cfg.dirs, gb, dt_code)
        bufs.append((bi, bo, torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)))
    s_in, s_cmp, s_out = (torch.cuda.Stream(dev) for _ in range(3))
    ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("in", "cmp", "out")}
    for k in ev:  # nothing pending on either buffer set at the start
        for e in ev[k]:
            e.record(torch.cuda.current_stream(dev))

    def step():
        for ci, (b, nb, g0) in enumerate(chunks):
            j = ci % 2
            bi0, bo0, wsj = bufs[j]
            bi = {n: view(v, nb) for n, v in bi0.items()}
            bo = {n: view(v, nb) for n, v in bo0.items()}
            s_in.wait_event(ev["cmp"][j])  # compute of chunk ci-2 has finished reading these inputs
            with torch.cuda.stream(s_in):
                for n in names:
                    for dst, src in zip(piece(bi[n], 0, nb, 0, n in wnames), piece(host_in[n], b, nb, g0, n in wnames)):
                        dst.copy_(src, non_blocking=True)
            ev["in"][j].record(s_in)
            s_cmp.wait_event(ev["in"][j])
            s_cmp.wait_event(ev["out"][j])  # D2H of chunk ci-2 has finished reading these outputs
            with torch.cuda.stream(s_cmp):
                gspn.fwd(bi["x"], bi["w_l"], bi["w_m"], bi["w_r"], bi["lam"], cfg.dirs, gb, out=bo["h"],
                         stream=s_cmp)
                gspn.bwd(bi["x"], bi["w_l"], bi["w_m"], bi["w_r"], bi["lam"], bo["h"], bi["dh"], cfg.dirs, gb,
                         outs=(bo["dx"], bo["dw_l"], bo["dw_m"], bo["dw_r"], bo["dlam"]), workspace=wsj,
                         stream=s_cmp)
            ev["cmp"][j].record(s_cmp)
            s_out.wait_event(ev["cmp"][j])
            with torch.cuda.stream(s_out):
                for n in onames:
                    for dst, src in zip(piece(host_out[n], b, nb, g0, n in wnames), piece(bo[n], 0, nb, 0, n in wnames)):
                        dst.copy_(src, non_blocking=True)
            ev["out"][j].record(s_out)

    main = torch.cuda.current_stream(dev)
    step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, args.e2e_steps)
    e0.record(main)
    for s_ in (s_in, s_cmp, s_out):
        s_.wait_event(e0)
    for _ in range(n):
        step()
    for s_ in (s_in, s_cmp, s_out):
        main.wait_stream(s_)
    e1.record(main)
    torch.cuda.synchronize(dev)
    ms = torch.tensor([e0.elapsed_time(e1) / n], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    total = (cfg.fwd_bytes() + cfg.bwd_bytes()) if args.scaling == "strong" else \
        (gspn.algorithmic_bytes(sh.B, sh.C, cfg.H, cfg.W, cfg.dirs, sh.G, dt_code, False) * 3 * world)
    return {"value": total / (ms * 1e-3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "ms_per_step": ms, "steps": n, "chunks": len(chunks),
            "note": "pinned host buffers; (b, group-block) chunks through 2 device buffer sets on 3 streams: "
                    "H2D of x,w,lam,dh | fwd + bwd | D2H of h,dx,dw,dlam overlap across chunks"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
