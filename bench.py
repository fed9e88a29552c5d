#!/usr/bin/env python
"""Benchmark of the GSPN line-scan hot path (fwd + bwd, all directions) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One "step" = one gspn_fwd + one gspn_bwd call (every SURVEY.md §8(a) row) over one batch of synthetic,
device-generated inputs already resident in HBM. Metric (BASELINE.json): algorithmic HBM GB/s of the
fwd+bwd scan, (bytes_fwd + bytes_bwd) / device time, bytes per SURVEY.md §8(d). Multi-GPU: one process
per GPU; `--gpus N` without a torchrun environment re-executes itself under torch.distributed.run with
N ranks. By default (--scaling strong) the ranks split ONE configuration: units (b, g) sharded
contiguously with no data-path collective, or -- for the single-unit config 5 -- channels, with the fp32
partial dw all-reduced over NCCL on a side stream (timed separately); --scaling weak gives every rank a
whole configuration (also measured and reported under `weak` at N > 1). The optional h all-gather
(north_star's "final output all-gather") is timed separately. Timing: CUDA events on the launching
stream, barrier + synchronize around the timed region, max over ranks; per-step median / p10 / p90.
At N = 1 the line also carries short runs of the other BASELINE configs (`configs`).

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
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the N ranks split one configuration; weak: one configuration per rank")
    ap.add_argument("--no-others", action="store_true",
                    help="skip the short runs of the other BASELINE configs reported under `configs` (N = 1)")
    ap.add_argument("--other-steps", type=int, default=10)
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
        g = oracle.bwd(sm["x"], *sm["ws"], sm["lam"], h, sm["dh"], sm["dirs"], 1, threads=sm["threads"])
        passes += 1
        wall = time.perf_counter() - t0
        if wall >= seconds:
            break
    last = {"h": h, "dx": g[0], "dw_l": g[1], "dw_m": g[2], "dw_r": g[3], "dlam": g[4]}
    return passes * sm["bytes"], wall, sm["threads"], f"{sm['desc']}; {passes} pass(es)", last


def oracle_sample(cfg, seconds: float):
    return oracle_time(oracle_prepare(cfg), seconds)[:4]


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
        b, w, threads, desc, _ = oracle_time(sm, per_step)
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

def pct(vals, q):
    v = sorted(vals)
    if not v:
        return None
    k = (len(v) - 1) * q
    lo, hi = int(k), min(int(k) + 1, len(v) - 1)
    return v[lo] + (v[hi] - v[lo]) * (k - lo)


def summary(vals):
    return {"median": pct(vals, 0.5), "p10": pct(vals, 0.1), "p90": pct(vals, 0.9)}


class Workload:
    """One rank's share of a configuration: device-generated inputs, outputs, workspace and the step."""

    def __init__(self, gspn, base, scaling, rank, world, dev, flags=0):
        import torch

        from synth.device import make_inputs, shard_for

        self.gspn, self.dev = gspn, dev
        self.base = base
        self.gcfg = base.with_(B=base.B * world) if scaling == "weak" else base
        self.sh = shard_for(self.gcfg, rank, world)
        sh, g = self.sh, self.gcfg
        self.t = make_inputs(g, dev, sh)
        self.dt_code = gspn.DTYPE_BF16 if g.dtype == "bf16" else gspn.DTYPE_F32
        # a single unit split by channel: each rank's dw is a partial sum over its channels, reduced in fp32
        self.channel_split = sh.kind == "channels"
        self.flags = flags | (gspn.FLAG_DW_F32 if self.channel_split else 0)
        self.h = torch.empty_like(self.t["lam"])
        if self.channel_split:
            self.dwbuf = torch.empty((3,) + tuple(self.t["w_l"].shape), dtype=torch.float32, device=dev)
            dw = (self.dwbuf[0], self.dwbuf[1], self.dwbuf[2])
        else:
            self.dwbuf = None
            dw = (torch.empty_like(self.t["w_l"]), torch.empty_like(self.t["w_m"]), torch.empty_like(self.t["w_r"]))
        self.outs = (torch.empty_like(self.t["x"]),) + dw + (torch.empty_like(self.t["lam"]),)
        wsb = gspn.workspace_bytes(sh.B, sh.C, g.H, g.W, g.dirs, sh.G, self.dt_code)
        self.ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
        self.bytes_f = gspn.algorithmic_bytes(sh.B, sh.C, g.H, g.W, g.dirs, sh.G, self.dt_code, False)
        self.bytes_b = gspn.algorithmic_bytes(sh.B, sh.C, g.H, g.W, g.dirs, sh.G, self.dt_code, True)
        self.work_bytes = sum(v.numel() * v.element_size() for v in self.t.values() if v is not None) + \
            self.h.numel() * self.h.element_size() + sum(o.numel() * o.element_size() for o in self.outs)
        self.launches = {"fwd": 0, "bwd": 0}
        self.paths = {"fwd": None, "bwd": None}

    def fwd(self):
        t, g = self.t, self.gcfg
        self.gspn.fwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], g.dirs, self.sh.G,
                      flags=self.flags & ~self.gspn.FLAG_DW_F32, out=self.h)
        self.launches["fwd"] = self.gspn.last_launch_count()
        self.paths["fwd"] = self.gspn.last_path()

    def bwd(self):
        t, g = self.t, self.gcfg
        self.gspn.bwd(t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"], self.h, t["dh"], g.dirs, self.sh.G,
                      flags=self.flags, outs=self.outs, workspace=self.ws)
        self.launches["bwd"] = self.gspn.last_launch_count()
        self.paths["bwd"] = self.gspn.last_path()

    def free(self):
        for k in list(self.__dict__):
            if k not in ("gspn", "dev", "base", "gcfg", "sh", "bytes_f", "bytes_b", "launches", "paths", "dt_code",
                         "channel_split", "flags", "work_bytes"):
                setattr(self, k, None)


def time_steps(wl, steps, warmup, stream, dev, world, dist, comm=None):
    """W untimed warm-up steps, then EXACTLY `steps` timed steps bracketed by barrier + synchronize.
    Per-step CUDA events on the launching stream: [start, fwd done, bwd done]; the config-5 fp32 dw
    all-reduce (channel split) runs on the side stream `comm`, overlapping the next step's fwd, and is
    timed there. Returns per-step lists (ms) and the region time (ms per step), max over ranks."""
    import torch

    flush = wl.work_bytes < 4 * L2_BYTES
    flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev) if flush else None
    comm_done = torch.cuda.Event()
    comm_done.record(stream)

    def step(evs=None):
        if evs:
            evs[0].record(stream)
        wl.fwd()
        if evs:
            evs[1].record(stream)
        stream.wait_event(comm_done)  # the previous step's reduction has read dw
        wl.bwd()
        if evs:
            evs[2].record(stream)
        if wl.channel_split:
            comm.wait_stream(stream)
            with torch.cuda.stream(comm):
                if evs:
                    evs[3].record(comm)
                dist.all_reduce(wl.dwbuf)  # fp32 partial dw, NCCL over NVLink
                if evs:
                    evs[4].record(comm)
            comm_done.record(comm)

    for _ in range(warmup):
        step()
        if flush:
            flush_buf.zero_()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    evs_all = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(5 if wl.channel_split else 3)]
        step(evs)
        evs_all.append(evs)
        if flush:
            flush_buf.zero_()
    if wl.channel_split:
        stream.wait_event(comm_done)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    f_ms = [e[0].elapsed_time(e[1]) for e in evs_all]
    b_ms = [e[1].elapsed_time(e[2]) for e in evs_all]
    c_ms = [e[3].elapsed_time(e[4]) for e in evs_all] if wl.channel_split else []
    region = ev0.elapsed_time(ev1) / steps
    vec = torch.tensor([region, pct(f_ms, 0.5), pct(b_ms, 0.5), pct(c_ms, 0.5) or 0.0], dtype=torch.float64,
                       device=dev)
    if world > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.MAX)
    region, fmed, bmed, cmed = [float(v) for v in vec.tolist()]
    return {"f": f_ms, "b": b_ms, "c": c_ms, "step": [a + b for a, b in zip(f_ms, b_ms)], "region": region,
            "f_med": fmed, "b_med": bmed, "c_med": cmed, "flush": flush}


def unit_slices(wl, n):
    """Host copies of the outputs of units (b, g) 0..n-1 (a full, unsharded workload), laid out like the
    oracle sample of `oracle_prepare` (units as the batch dimension, C/G channels, G = 1)."""
    import torch

    g = wl.gcfg
    Cg = g.C // g.G
    h, (dx, dwl, dwm, dwr, dlam) = wl.h, wl.outs
    out = {k: [] for k in ("h", "dx", "dw_l", "dw_m", "dw_r", "dlam")}
    for u in range(n):
        b, gr = divmod(u, g.G)
        c0 = gr * Cg
        out["h"].append(h[:, b, c0:c0 + Cg])
        out["dlam"].append(dlam[:, b, c0:c0 + Cg])
        out["dx"].append(dx[b, c0:c0 + Cg])
        for name, t in (("dw_l", dwl), ("dw_m", dwm), ("dw_r", dwr)):
            out[name].append(t[:, b, gr:gr + 1])
    res = {}
    for k, v in out.items():
        st = torch.stack(v, dim=0 if k == "dx" else 1)
        res[k] = st.to(torch.float64).cpu().numpy()
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2512_07884_b200 as gspn
    from synth.configs import get_config

    rank, world, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime

        # NCCL failures (a dead peer, a hung collective) abort the process group instead of hanging the job
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(minutes=5))

    base = get_config(args.config)
    if args.dirs is not None:
        base = base.with_(dirs=args.dirs)
    wl = Workload(gspn, base, args.scaling, rank, world, dev, args.flags)
    gcfg, sh = wl.gcfg, wl.sh
    stream = torch.cuda.current_stream(dev)
    comm = torch.cuda.Stream(dev) if wl.channel_split else None

    clocks = ClockSampler(local)
    clocks.start()
    t_wall0 = time.perf_counter()
    tm = time_steps(wl, args.steps, args.warmup, stream, dev, world, dist, comm)
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    launches = dict(wl.launches)
    paths = dict(wl.paths)
    total_bytes = gcfg.fwd_bytes() + gcfg.bwd_bytes()  # the whole job (all ranks)
    # the timed region; when L2 is flushed between steps (small configs) the flush memsets sit inside it, so
    # the step is then the sum of the per-call event medians (max over ranks)
    step_ms = tm["f_med"] + tm["b_med"] if tm["flush"] else tm["region"]
    # per-unit parity sample of this run's outputs (compared with the oracle in the cpu_baseline leg)
    par_units = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        par_units = unit_slices(wl, min(2, gcfg.B * gcfg.G))

    # ---- N > 1: the h all-gather (north_star "final output all-gather"), timed separately
    weak, allgather = None, None
    if world > 1:
        hsz = wl.h.numel()
        full = torch.empty(hsz * world, dtype=wl.h.dtype, device=dev)
        ag = []
        for i in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dist.all_gather_into_tensor(full, wl.h.reshape(-1))
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if i:
                ag.append(e0.elapsed_time(e1))
        agv = torch.tensor([pct(ag, 0.5)], dtype=torch.float64, device=dev)
        dist.all_reduce(agv, op=dist.ReduceOp.MAX)
        nbytes = full.numel() * full.element_size()
        allgather = {"ms": float(agv.item()), "bytes_total": nbytes,
                     "note": "h [D,B,C,H,W] shards gathered to every rank (rank-major), NCCL, outside `value`"}
        del full
    # ---- SURVEY §8(f) rows on the same workload (after the headline region; not part of `value`)
    nxt = None
    if not args.no_next and world == 1:
        nxt = measure_next(args, gspn, gcfg, sh, wl.t, wl.h, wl.outs, wl.ws, dev, stream)

    # ---- end to end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and wl.t is not None:
        e2e = run_e2e(args, gspn, gcfg, sh, wl.t, wl.h, wl.outs, wl.ws, dev, world, dist)
    if wl.t is not None:
        wl.free()
        torch.cuda.empty_cache()

    if world > 1:
        if args.scaling == "strong":
            ww = Workload(gspn, base, "weak", rank, world, dev, args.flags)
            tw = time_steps(ww, args.steps, args.warmup, stream, dev, world, dist,
                            torch.cuda.Stream(dev) if ww.channel_split else None)
            wb = ww.gcfg.fwd_bytes() + ww.gcfg.bwd_bytes()
            weak = {"value": wb / (tw["region"] * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": tw["region"],
                    "config": f"{world} x config {base.name} (B={ww.gcfg.B})"}
            ww.free()

    # ---- the other BASELINE configs, short runs on the same device (N = 1 only)
    others = None
    if world == 1 and not args.no_others:
        others = measure_others(args, gspn, base.name, dev, stream)

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sm = oracle_prepare(base)
            b_cpu, w_cpu, thr, desc, last = oracle_time(sm, args.cpu_seconds)
            cpu = {"value": b_cpu / w_cpu / 1e9, "unit": "GB/s", "cores": thr, "kind": "oracle", "sample": desc}
            parity = parity_vs_oracle(par_units, last, gcfg.dtype)
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0
    peak, peak_src = peaks()
    mean_f, mean_b = tm["f_med"], tm["b_med"]
    bytes_f, bytes_b = wl.bytes_f, wl.bytes_b
    dominant = "bwd" if mean_b >= mean_f else "fwd"
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
            "per_rank": {"B": sh.B, "C": sh.C, "G": sh.G, "kind": sh.kind, "units": sh.units,
                         "fwd_bytes": bytes_f, "bwd_bytes": bytes_b},
            "fwd_ms": mean_f, "bwd_ms": mean_b,
            "step_ms": summary(tm["step"]), "fwd_ms_pct": summary(tm["f"]), "bwd_ms_pct": summary(tm["b"]),
            "fwd_gbs": bytes_f / (mean_f * 1e-3) / 1e9, "bwd_gbs": bytes_b / (mean_b * 1e-3) / 1e9,
            "algorithmic_bytes_per_step": total_bytes,
            "l2": ("L2 flushed (2x126 MB memset) between steps, outside the event pairs" if tm["flush"] else
                   f"inputs+outputs {wl.work_bytes / 1e9:.1f} GB > 126 MB L2, no flush"),
            "path": paths,
            "wall_s_timed_region": t_wall,
        },
        "roofline": {
            "bound": "hbm", "kernel": f"gspn_{dominant} ({paths[dominant]} path, {launches[dominant]} launch(es))",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": peak_src,
            "traffic": traffic_for(base.name, dominant) if world == 1 else None,
            "algorithmic_bytes_per_launch": dom_bytes,
            "step_frac": value / world / peak,
        },
        "clocks": clk,
        "gpu_launches": args.steps * (launches["fwd"] + launches["bwd"]),
        "launches_per_call": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
        "next": nxt,
        "configs": others,
    }
    if wl.channel_split:
        line["collective"] = {"dw_allreduce_ms": tm["c_med"], "dtype": "f32",
                              "bytes": 3 * gcfg.D * gcfg.H * gcfg.W * 4,
                              "note": "NCCL all-reduce of the fp32 partial dw on a side stream; overlaps the next "
                                      "step's fwd, completes inside the timed region"}
    if weak is not None:
        line["weak"] = weak
    if allgather is not None:
        line["h_allgather"] = allgather
    print(json.dumps(line), flush=True)
    return 0


def parity_vs_oracle(gpu, ref, dtype):
    """normwise max|gpu - ref| / max|ref| per output (R16) on the first units of the headline
    run vs the oracle's last pass over the same units (its own unrounded h: end to end)."""
    if gpu is None or ref is None:
        return None
    import numpy as np

    n = gpu["h"].shape[1]
    out = {"units": n, "tol": 1e-5 if dtype == "f32" else 2e-2, "kind": "normwise, end to end vs fp64 oracle"}
    for k in ("h", "dx", "dw_l", "dw_m", "dw_r", "dlam"):
        r = ref[k][:n] if k == "dx" else ref[k][:, :n]
        g = gpu[k].reshape(r.shape)
        den = float(np.abs(r).max())
        out[k] = float(np.abs(g - r).max() / den) if den > 0 else 0.0
    return out


def measure_others(args, gspn, skip, dev, stream):
    """Short device-timed runs (one GPU, full configuration) of the other BASELINE configs, so every
    config gets a driver-measured line: median / p10 / p90 step time, GB/s, fraction of the peak."""
    import torch

    from synth.configs import CONFIGS

    peak, _ = peaks()
    res = {}
    for name, cfg in CONFIGS.items():
        if name == skip:
            continue
        try:
            wl = Workload(gspn, cfg, "strong", 0, 1, dev)
            tm = time_steps(wl, max(3, args.other_steps), max(3, args.warmup), stream, dev, 1, None)
            tb = cfg.fwd_bytes() + cfg.bwd_bytes()
            # flushed runs: the region also holds the L2 flushes, so the step is timed by its own events
            ms = pct(tm["step"], 0.5) if tm["flush"] else tm["region"]
            gbs = tb / (ms * 1e-3) / 1e9
            res[name] = {"ms_per_step": ms, "step_ms": summary(tm["step"]), "fwd_ms": tm["f_med"],
                         "bwd_ms": tm["b_med"], "value": gbs, "unit": "GB/s", "frac": gbs / peak,
                         "path": dict(wl.paths), "launches_per_call": dict(wl.launches),
                         "l2": "flushed between steps" if tm["flush"] else "working set > 4x L2"}
            wl.free()
            del wl
            torch.cuda.empty_cache()
        except Exception as ex:
            res[name] = {"error": str(ex)}
    return res


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
    # NEXT-1 fused: the scan's backward through the merge in one launch (dh = s u dy never stored), and the
    # forward + merge in one cooperative launch; vs the unfused chain fwd, merge_fwd, merge_bwd, bwd
    wsm = torch.empty(max(16, int(gspn.lib().gspn_bwd_merged_workspace_bytes(sh.B, sh.C, cfg.H, cfg.W, cfg.dirs, sh.G,
                                                                               gspn.DTYPE_BF16 if cfg.dtype == "bf16"
                                                                               else gspn.DTYPE_F32))),
                      dtype=torch.uint8, device=dev)
    a = (t["x"], t["w_l"], t["w_m"], t["w_r"], t["lam"])
    fm = timed(lambda: gspn.fwd_merged(*a, u, cfg.dirs, sh.G, out=y, h_out=h), reps)
    pfm = (gspn.last_path(), gspn.last_launch_count())
    bm = timed(lambda: gspn.bwd_merged(*a, h, u, dy, cfg.dirs, sh.G, outs=tuple(outs) + (du,), workspace=wsm), reps)
    pbm = (gspn.last_path(), gspn.last_launch_count())
    f0 = timed(lambda: gspn.fwd(*a, cfg.dirs, sh.G, out=h), reps)
    b0 = timed(lambda: gspn.bwd(*a, h, dh2, cfg.dirs, sh.G, outs=outs, workspace=ws), reps)
    # NEXT-3: checkpointing forward (no h) + recompute backward vs the saved-h step
    if cfg.G == cfg.C:
        ckb = int(gspn.lib().gspn_ckpt_bytes(sh.B, sh.C, cfg.H, cfg.W, cfg.dirs, sh.G,
                                             gspn.DTYPE_BF16 if cfg.dtype == "bf16" else gspn.DTYPE_F32))
        ck = torch.empty(max(4, ckb // 4), dtype=torch.float32, device=dev)
        wsr = torch.empty(max(16, int(gspn.lib().gspn_bwd_recompute_workspace_bytes(
            sh.B, sh.C, cfg.H, cfg.W, cfg.dirs, sh.G, gspn.DTYPE_BF16 if cfg.dtype == "bf16" else gspn.DTYPE_F32))),
            dtype=torch.uint8, device=dev)
        fc = timed(lambda: gspn.fwd_ckpt(*a, cfg.dirs, sh.G, ckpt=ck), reps)
        pfc = (gspn.last_path(), gspn.last_launch_count())
        br = timed(lambda: gspn.bwd_recompute(*a, ck, t["dh"], cfg.dirs, sh.G, outs=outs, workspace=wsr), reps)
        pbr = (gspn.last_path(), gspn.last_launch_count())
        b_s = timed(lambda: gspn.bwd(*a, h, t["dh"], cfg.dirs, sh.G, outs=outs, workspace=ws), reps)
        out["recompute"] = {"fwd_ckpt_ms": fc, "fwd_ckpt_path": pfc, "bwd_recompute_ms": br, "bwd_recompute_path": pbr,
                            "step_ms": fc + br, "saved_h_step_ms": f0 + b_s, "ckpt_bytes": ckb,
                            "note": "fwd writes fp32 checkpoints every half-tile instead of h; the bwd recomputes h "
                                    "in registers and forms every direction's dw in the recurrence"}
        del ck, wsr
    out["merged_step"] = {"fwd_merged_ms": fm, "fwd_merged_path": pfm, "bwd_merged_ms": bm, "bwd_merged_path": pbm,
                          "fused_step_ms": fm + bm, "unfused_step_ms": f0 + mf + mb + b0,
                          "unfused": {"fwd": f0, "merge_fwd": mf, "merge_bwd": mb, "bwd": b0}}
    del wsm
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
    # NEXT-4: proxy projections (gspn_proxy_mix / _wgrad) on the compact blocks of BASELINE configs[2]
    # (B=64, C=384 -> C_proxy=8, 28 x 28) and configs[4] (B=1, C=320 -> 40, 2048 x 2048): tcgen05 path
    # (default for bf16) and the SIMT kernel; bytes = s B HW (C + C_proxy) per mix / wgrad.
    dtp = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(7884)
    out["proxy"] = {}
    for tag, (pB, pC, pCp, pH, pW) in (("cfg3", (64, 384, 8, 28, 28)), ("cfg5", (1, 320, 40, 2048, 2048))):
        xin = (torch.rand((pB, pC, pH, pW), generator=g, device=dev) * 2 - 1).to(dtp)
        Pd = ((torch.rand((pCp, pC), generator=g, device=dev) * 2 - 1) / pC ** 0.5).to(dtp)
        Qu = ((torch.rand((pC, pCp), generator=g, device=dev) * 2 - 1) / pCp ** 0.5).to(dtp)
        xp = torch.empty((pB, pCp, pH, pW), dtype=dtp, device=dev)
        yo = torch.empty_like(xin)
        dPd = torch.empty((pCp, pC), dtype=torch.float32, device=dev)
        nb = 2 * pB * pH * pW * (pC + pCp)
        rec = {"shape": f"B={pB} C={pC} C_proxy={pCp} {pH}x{pW} bf16", "bytes": nb}
        for impl, simt in (("umma", False), ("simt", True)):
            md = timed(lambda: gspn.proxy_mix(xin, Pd, out=xp, simt=simt), reps)
            pth = gspn.last_path()
            mu = timed(lambda: gspn.proxy_mix(xp, Qu, out=yo, simt=simt), reps)
            rec[impl] = {"path": pth, "down_ms": md, "down_gbs": nb / (md * 1e-3) / 1e9, "down_frac": nb / (md * 1e-3) / 1e9 / peak,
                         "up_ms": mu, "up_gbs": nb / (mu * 1e-3) / 1e9, "up_frac": nb / (mu * 1e-3) / 1e9 / peak}
        mw = timed(lambda: gspn.proxy_wgrad(xp, xin, out=dPd), reps)
        rec["wgrad"] = {"path": gspn.last_path(), "ms": mw, "gbs": nb / (mw * 1e-3) / 1e9, "frac": nb / (mw * 1e-3) / 1e9 / peak}
        out["proxy"][tag] = rec
        del xin, Pd, Qu, xp, yo, dPd
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


def maybe_spawn(args):
    """`--gpus N` outside torchrun: re-execute under torch.distributed.run with N ranks on this node."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
