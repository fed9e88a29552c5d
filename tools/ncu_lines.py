"""Summarise an ncu 'source --print-source cuda,sass' CSV: per source line, instructions executed and
stall samples (top N). Usage: python tools/ncu_lines.py file.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None
hdr = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split('/')[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samples = int(r[4]) if r[4] not in ("-", "") else 0
        inst = int(r[7]) if r[7] not in ("-", "") else 0
    except (ValueError, IndexError):
        continue
    out.append((samples, inst, cur_file, r[0], r[1].strip()[:110]))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s}  total warp-inst {tot_i}")
for s, i, f, ln, src in sorted(out, reverse=True)[:N]:
    print(f"{100*s/tot_s:5.1f}%s {100*i/tot_i:5.1f}%i  {f}:{ln:5s} {src}")
