"""Split an ncu SASS source page (csv) by called function: executed
instructions, stall samples, FP64 share per function body.
usage: python tools/ncu_funcsplit.py source.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
ins = []
for d in data:
    try:
        a = int(d["Address"], 16)
    except ValueError:
        continue
    ins.append((a, d["Source"], float(d["Instructions Executed"] or 0), float(d["Warp Stall Sampling (All Samples)"] or 0)))
ins.sort()
targets = sorted({int(m.group(1), 16) for _, s, _, _ in ins for m in [re.search(r"CALL\.\S+\s+0x([0-9a-f]+)", s)] if m})
bounds = [ins[0][0]] + targets + [1 << 62]
tot_e = sum(e for _, _, e, _ in ins) or 1
tot_s = sum(s for _, _, _, s in ins) or 1
print(f"{'start':>14} {'#ins':>6} {'exec%':>6} {'samp%':>6} {'fp64%':>6}  top ops")
for lo, hi in zip(bounds, bounds[1:]):
    seg = [x for x in ins if lo <= x[0] < hi]
    if not seg:
        continue
    e = sum(x[2] for x in seg)
    s = sum(x[3] for x in seg)
    ops = defaultdict(float)
    for _, src, ex, _ in seg:
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].split(".")[0] if src.strip() else "?"
        ops[op] += ex
    fp = sum(v for k, v in ops.items() if k in ("DADD", "DMUL", "DFMA", "DSETP")) / (e or 1)
    top = sorted(ops.items(), key=lambda t: -t[1])[:6]
    print(f"{lo:#14x} {len(seg):6d} {100*e/tot_e:6.1f} {100*s/tot_s:6.1f} {100*fp:6.1f}  " + " ".join(f"{k}:{100*v/(e or 1):.0f}" for k, v in top))
