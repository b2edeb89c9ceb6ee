"""Per-phase instruction / stall shares of search_kernel from an ncu source dump
(tools/ncu_summary.sh writes /tmp/_ncu_src.csv). Phases are line ranges of
one source file given as name=lo-hi arguments; other files are reported apart.

  python tools/phase_hot.py /tmp/_ncu_src.csv search.cu eval=80-140 ..."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
phases = []
target = sys.argv[2]
for a in sys.argv[3:]:
    name, rng = a.split("=")
    lo, hi = map(int, rng.split("-"))
    phases.append((name, lo, hi))
cur_file, hdr, cur_line = None, None, None
st, ex = defaultdict(int), defaultdict(int)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:
        cur_line = (cur_file, int(r[0]))
    try:
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        e = int(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    st[cur_line] += s
    ex[cur_line] += e
ts, te = sum(st.values()) or 1, sum(ex.values()) or 1
agg_s, agg_e = defaultdict(int), defaultdict(int)
for (f, ln), e in ex.items():
    name = f
    if f == target:
        for p, lo, hi in phases:
            if lo <= ln <= hi:
                name = p
                break
    agg_e[name] += e
    agg_s[name] += st[(f, ln)]
for name in sorted(agg_e, key=lambda k: -agg_e[k]):
    print(f"{name:24s} inst {100 * agg_e[name] / te:5.1f}%  stall {100 * agg_s[name] / ts:5.1f}%")
