"""Dev: split an ncu SASS source page (csv) into functions (CALL targets),
and print per-function executed instructions, stall samples and opcode mix.
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_funcs.py x.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
addr = [int(d["Address"], 16) for d in data]
targets = {addr[0]}
for d in data:
    m = re.search(r"CALL\.\w+(?:\.\w+)* (0x[0-9a-f]+)", d["Source"])
    if m:
        targets.add(int(m.group(1), 16))
starts = sorted(targets)
def fid(a):
    lo = 0
    for i, s in enumerate(starts):
        if s <= a:
            lo = i
    return lo
agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), 0])
tot_i = tot_s = 0
for d, a in zip(data, addr):
    f = fid(a)
    ie = int(d["Instructions Executed"] or 0)
    ss = int(d["Warp Stall Sampling (All Samples)"] or 0)
    op = d["Source"].split()
    op = (op[1] if op and op[0].startswith("@") else (op[0] if op else "")).split(".")[0]
    agg[f][0] += ie
    agg[f][1] += ss
    agg[f][2][op] += ie
    agg[f][3] += 1
    tot_i += ie
    tot_s += ss
print(f"total executed {tot_i}, samples {tot_s}")
for f in sorted(agg, key=lambda k: -agg[k][1]):
    ie, ss, ops, n = agg[f]
    if ss < 0.005 * tot_s:
        continue
    mix = ", ".join(f"{o} {100 * c / max(ie, 1):.0f}%" for o, c in ops.most_common(6))
    print(f"f{f:02d} @{starts[f]:#x} size {n:5d}  instr {100 * ie / tot_i:5.1f}%  samples {100 * ss / tot_s:5.1f}%  | {mix}")
