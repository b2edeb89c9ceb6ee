"""Summarise an ncu --page source --csv (SASS) dump: hottest instructions by
stall samples and executed count, plus totals per instruction class."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = col["Warp Stall Sampling (All Samples)"]
E = col["Instructions Executed"]
tot_s = sum(int(r[S] or 0) for r in data)
tot_e = sum(int(r[E] or 0) for r in data)
print(f"instructions {len(data)}, stall samples {tot_s}, warp instructions executed {tot_e}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
idx = sorted(range(len(data)), key=lambda i: -int(data[i][S] or 0))[:top]
for i in sorted(idx):
    r = data[i]
    print(f"{i:5d} {int(r[S] or 0):7d} {100*int(r[S] or 0)/tot_s:5.1f}% exec={int(r[E] or 0):10d}  {r[col['Source']].strip()}")
ops = Counter()
for r in data:
    op = r[col["Source"]].strip().split()[0] if r[col["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[col["Source"]].strip().split()[1]
    ops[op.split(".")[0]] += int(r[E] or 0)
print("executed by opcode:", ", ".join(f"{k}:{v/tot_e:.1%}" for k, v in ops.most_common(18)))
