"""Per-opcode instruction mix from an ncu source CSV exported with --print-source cuda,sass
(rows with a SASS address). Also prints the hottest SASS instructions by executed count.

  ncu -i rep --page source --csv --print-source cuda,sass --kernel-name regex:K > k.csv
  python tools/ncu_ops.py k.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ops = collections.Counter()
samp = collections.Counter()
hot = {}
for r in rows:
    if len(r) < 8 or not r[2].startswith("0x"):
        continue
    try:
        inst = int(r[7])
        s = int(r[4])
    except ValueError:
        continue
    text = r[3].strip()
    tok = text.split()
    if not tok:
        continue
    op = tok[1] if tok[0].startswith("@") else tok[0]
    ops[op.split(".")[0]] += inst
    samp[op.split(".")[0]] += s
    hot[r[2]] = (inst, s, text)
tot = sum(ops.values()) or 1
ts = sum(samp.values()) or 1
print(f"total warp-inst {tot}")
for op, n in ops.most_common(N):
    print(f"{100 * n / tot:5.1f}%i {100 * samp[op] / ts:5.1f}%s  {op}")
print("-- hottest instructions")
for a, (n, s, t) in sorted(hot.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{n:>12} {s:>6}  {t[:90]}")
