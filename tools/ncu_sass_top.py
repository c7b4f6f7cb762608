"""Summarise an `ncu --page source --csv` SASS dump: top instructions by
stall samples and by executed count (usage: ncu_sass_top.py file.csv [N])."""
import csv
import sys

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
with open(path) as f:
    rows = list(csv.reader(f))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
num = lambda x: float(x) if x not in ("", None) else 0.0
ks, ki = "Warp Stall Sampling (All Samples)", "Instructions Executed"
ts = sum(num(d[ks]) for d in data) or 1
ti = sum(num(d[ki]) for d in data) or 1
print(f"instructions: {len(data)}  samples {ts:.0f}  warp-instr executed {ti:.0f}")
for i, d in enumerate(data):
    d["idx"] = i
print("--- by stall samples")
for d in sorted(data, key=lambda d: -num(d[ks]))[:N]:
    print(f"{d['idx']:5d} {d['Address']:>6} s={num(d[ks]) / ts * 100:5.2f}% i={num(d[ki]) / ti * 100:5.2f}%  {d['Source'][:100]}")
# opcode histogram weighted by executed count
from collections import Counter
c = Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    c[op.split(".")[0]] += num(d[ki])
print("--- opcode mix (executed)")
for op, v in c.most_common(25):
    print(f"{op:12s} {v / ti * 100:5.1f}%")
print("--- by executed count")
for d in sorted(data, key=lambda d: -num(d[ki]))[:N]:
    print(f"{d['idx']:5d} s={num(d[ks]) / ts * 100:5.2f}% i={num(d[ki]) / ti * 100:5.2f}%  {d['Source'][:100]}")
