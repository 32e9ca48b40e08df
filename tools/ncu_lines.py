"""Warp-stall samples and executed instructions per CUDA source line of one ncu report.
usage: ncu -i REP --page source --csv --print-source cuda,sass > /tmp/src.csv; python tools/ncu_lines.py /tmp/src.csv [top]"""
import csv
import sys
from collections import defaultdict


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
agg = defaultdict(lambda: [0.0, 0.0])
src = {}
for r in rows:
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9 or not r[0]:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    src[ln] = r[1]
    agg[ln][0] += num(r[4])
    agg[ln][1] += num(r[7])
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot:.0f}, warp instructions {toti:.3e}")
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% stall  {100 * v[1] / toti:5.1f}% inst  {ln:5d} {src[ln][:90]}")
