"""Write profiles/traffic.json (DRAM bytes per fwd / bwd call, the bench roofline's `traffic`) from one
`ncu --set full` capture of the bench command (tools/profile.sh).

  python tools/traffic_json.py gpurun_out/prof_cfg4.ncu-rep --config 4 --source profiles/r1_cfg4_ncu.md
"""
import argparse
import csv
import io
import json
import os
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--config", default="4")
ap.add_argument("--source", default=None)
ap.add_argument("--out", default=os.path.join(os.path.dirname(__file__), "..", "profiles", "traffic.json"))
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
ki = hdr.index("Kernel Name")
col = {m: hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
units = rows[1]


def val(r, m):
    v = float(r[col[m]].replace(",", ""))
    u = units[col[m]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    return v * scale.get(u, 1)


calls = {"fwd": 0.0, "bwd": 0.0}
kernels = []
for r in rows[2:]:
    name = r[ki]
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    t = val(r, "gpu__time_duration.sum")
    call = "fwd" if "fwd_" in name else ("bwd" if ("bwd_" in name or "out_" in name) else None)
    if call is None:
        continue
    calls[call] += b
    kernels.append({"kernel": name.split("(")[0], "call": call, "dram_bytes": b, "ms": t})
try:
    data = json.load(open(a.out))
except Exception:
    data = {}
data[a.config] = {"fwd": calls["fwd"], "bwd": calls["bwd"], "unit": "bytes per call (DRAM read + write)",
                  "kernels": kernels, "source": a.source or a.rep}
json.dump(data, open(a.out, "w"), indent=1)
print(json.dumps(data[a.config], indent=1))
