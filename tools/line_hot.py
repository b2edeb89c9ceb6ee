"""Aggregate an ncu '--page source --csv --print-source cuda,sass' dump per CUDA
source line: stall samples and warp instructions executed."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
stalls = defaultdict(int)
execs = defaultdict(int)
text = {}
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None:
        continue
    if r[0]:
        cur_line = (cur_file, int(r[0]))
        text[cur_line] = r[1].strip()
    try:
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        e = int(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    stalls[cur_line] += s
    execs[cur_line] += e
ts = sum(stalls.values()) or 1
te = sum(execs.values()) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"stall samples {ts}, warp instructions {te}")
for key in sorted(stalls, key=lambda k: -stalls[k])[:top]:
    print(f"{key[0]}:{key[1]:<5d} stall {100*stalls[key]/ts:5.1f}%  inst {100*execs[key]/te:5.1f}%  {text.get(key, '')[:90]}")
