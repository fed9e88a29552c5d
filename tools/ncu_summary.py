"""Summarise an ncu report (.ncu-rep) into markdown: per kernel, duration, DRAM bytes vs algorithmic,
throughput, occupancy, shared-memory bank conflicts, L2 hit rate and the top stall reasons.

  python tools/ncu_summary.py gpurun_out/prof_cfg4.ncu-rep [--alg fwd=14.0929e9 --alg bwd=28.1857e9]
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "GPU DRAM throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem, CTAs)"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs, CTAs)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw_rows(rep: str):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--alg", action="append", default=[], help="kernel-substring=algorithmic bytes per launch")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    alg = {}
    for s in a.alg:
        k, v = s.split("=")
        alg[k] = float(v)
    hdr, units, rows = raw_rows(a.rep)
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu summary {a.title}\n\nsource: `{a.rep}` (ncu --set full --clock-control none)\n")
    for r in rows:
        name = r[idx["Kernel Name"]]
        print(f"## `{name}`\n")
        print("| metric | value |\n|---|---|")
        vals = {}
        for m, label in METRICS:
            if m in idx:
                v = r[idx[m]]
                vals[m] = v
                print(f"| {label} (`{m}`) | {v} {units[idx[m]]} |")
        try:
            rd = float(vals["dram__bytes_read.sum"]) * (1e9 if "Gbyte" in units[idx["dram__bytes_read.sum"]] else
                                                      1e6 if "Mbyte" in units[idx["dram__bytes_read.sum"]] else 1)
            wr = float(vals["dram__bytes_write.sum"]) * (1e9 if "Gbyte" in units[idx["dram__bytes_write.sum"]] else
                                                       1e6 if "Mbyte" in units[idx["dram__bytes_write.sum"]] else 1)
            for k, v in alg.items():
                if k in name:
                    print(f"| DRAM traffic / algorithmic bytes | {(rd + wr) / v:.3f} ({(rd + wr) / 1e9:.3f} GB / "
                          f"{v / 1e9:.3f} GB) |")
        except (KeyError, ValueError):
            pass
        stalls = []
        for h, i in idx.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = sorted(stalls, reverse=True)[:8]
        print("\nTop stall reasons (share of PC samples): " +
              ", ".join(f"{n} {100 * s / tot:.1f}%" for s, n in top) + "\n")


if __name__ == "__main__":
    main()
