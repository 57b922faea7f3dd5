"""Warp-stall samples per CUDA source line from `ncu --page source --csv --print-source cuda,sass`.
usage: python tools/ncu_lines.py file.csv [top]"""
import collections
import csv
import sys

agg, src, cur, idx = collections.Counter(), {}, None, None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        idx = {c: i for i, c in enumerate(r)}
        continue
    if idx is None or not r[0].isdigit() or r[2].startswith("0x"):
        continue
    try:
        v = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        v = 0.0
    agg[(cur, int(r[0]))] += v
    src[(cur, int(r[0]))] = r[1].strip()[:90]
T = sum(agg.values()) or 1.0
print("total samples", T)
for (f, ln), v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{v:8.0f} {100 * v / T:5.1f}% {f}:{ln} {src[(f, ln)]}")
