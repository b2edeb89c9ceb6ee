"""Top SASS instructions of an ncu '--page source --csv --print-source sass' dump
by stall samples, with the dominant stall reasons and execution counts.

  python tools/sass_stalls.py /tmp/sass.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = {h: i for i, h in enumerate(rows[1])}
reasons = [h for h in rows[1] if h.startswith("stall_") and "Not Issued" not in h]
data = []
for idx, r in enumerate(rows[2:]):
    try:
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        e = int(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    rs = {h: int(r[hdr[h]] or 0) for h in reasons}
    data.append((idx, r[1].strip(), s, e, rs))
ts = sum(d[2] for d in data) or 1
te = sum(d[3] for d in data) or 1
tot = {h: sum(d[4][h] for d in data) for h in reasons}
print(f"samples {ts} instructions {te}")
print("mix:", ", ".join(f"{h[6:]} {100 * v / ts:.1f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for idx, txt, s, e, rs in sorted(data, key=lambda d: -d[2])[:top]:
    why = ", ".join(f"{h[6:]}:{100 * v / max(1, s):.0f}" for h, v in sorted(rs.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{idx:5d} {100 * s / ts:5.2f}% exec {e / 1e6:7.2f}M  {txt[:60]:60s} {why}")
