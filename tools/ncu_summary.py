"""Summarise an ncu SASS source page (csv): stall reasons totals, top instructions.
usage: ncu -i rep --page source --csv > x.csv; python tools/ncu_summary.py x.csv [topN]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for d in data:
    for s in stalls:
        tot[s] += f(d[s])
allsamp = sum(tot.values()) or 1
print("stall totals (% of samples):")
for s, v in tot.most_common(12):
    print(f"  {s:28s} {100 * v / allsamp:5.1f}%")
ops = Counter()
execd = Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"] else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    ops[op.split(".")[0]] += f(d["Warp Stall Sampling (All Samples)"])
    execd[op.split(".")[0]] += f(d["Instructions Executed"])
te = sum(execd.values()) or 1
print("executed warp instructions by opcode:")
for o, v in execd.most_common(20):
    print(f"  {o:10s} {100 * v / te:5.1f}%  stall-samples {100 * ops[o] / allsamp:5.1f}%")
print("top instructions by stall samples:")
data.sort(key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))
for d in data[:top]:
    reasons = sorted(((f(d[s]), s) for s in stalls), reverse=True)[:2]
    print(f"  {100 * f(d['Warp Stall Sampling (All Samples)']) / allsamp:5.2f}% {d['Address']} "
          f"{d['Source'][:60]:60s} {reasons}")
