"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
total device time per kernel name and its share."""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if "Kernel Name" in r)
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    name = re.sub(r"gann::(\(anonymous namespace\)::)?", "", name)
    v = float(r[vi].replace(",", ""))
    unit = r[unit_i] if unit_i is not None else "ns"
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.1f} ms over {sum(cnt.values())} launches")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{tot[k]:10.2f} ms {100*tot[k]/T:5.1f}%  x{cnt[k]:<5d} {k}")
