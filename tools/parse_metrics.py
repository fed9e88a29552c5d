"""Print per-kernel duration / DRAM bytes from `ncu --metrics ... --csv` outputs.

  python tools/parse_metrics.py gpurun_out/exp_*.csv
"""
import csv
import sys


def parse(path):
    rows = list(csv.reader(open(path)))
    d = {}
    for r in rows:
        if len(r) < 15 or not r[0].isdigit():
            continue
        name = r[4]
        k = "fwd" if "fwd_stream" in name else ("bwd" if "bwd_stream" in name else ("out" if "out_" in name else name[:30]))
        d.setdefault((int(r[0]), k), {})[r[12]] = (r[13], r[14])
    out = []
    for (i, k), m in sorted(d.items()):
        def val(key):
            u, v = m[key]
            return float(v.replace(",", "")), u
        t, _ = val("gpu__time_duration.sum")
        rd, _ = val("dram__bytes_read.sum")
        wr, _ = val("dram__bytes_write.sum")
        out.append(f"{k} {t / 1e6:.3f} ms  read {rd / 1e9:.2f} GB  write {wr / 1e9:.2f} GB")
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        for line in parse(p):
            print("   " + line)
