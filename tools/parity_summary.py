"""Summarise a $GSPN_ERRLOG JSON-lines file (measured normwise errors of the GPU parity tests) into markdown:
the worst error per test family and tensor, its tolerance and margin. Usage: python tools/parity_summary.py LOG"""
import json
import re
import sys

worst = {}
n = 0
for line in open(sys.argv[1]):
    d = json.loads(line)
    n += 1
    fam = re.sub(r"\[.*", "", d["test"].split("::")[-1])
    key = (fam, d["tensor"], d["tol"])
    if key not in worst or d["normwise"] > worst[key][0]:
        worst[key] = (d["normwise"], d["test"].split("::")[-1])
print(f"{n} recorded errors; worst per test family, tensor and tolerance (normwise = max|got - ref| / max|ref|)\n")
print("| test | tensor | tol | worst normwise | margin (tol / err) | worst case |")
print("|---|---|---|---|---|---|")
for (fam, t, tol), (e, case) in sorted(worst.items()):
    m = f"{tol / e:.1f}x" if e > 0 else "exact"
    print(f"| {fam} | {t} | {tol:g} | {e:.3e} | {m} | `{case[:70]}` |")
