"""Aggregate ncu warp-stall samples per CUDA source line (ncu --page source --csv --print-source cuda,sass)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(float)
src = {}
fname = "?"
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        continue
    if len(r) > 4:
        if r[0].strip():
            line = (fname, int(r[0]))
            src[line] = r[1].strip()
        try:
            v = float(r[4] or 0)
        except ValueError:
            continue
        if line is not None:
            agg[line] += v
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]:<5} {src.get(k, '')[:100]}")
