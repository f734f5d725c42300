"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export per
CUDA source line: share of warp-stall samples and executed instructions.
Usage: python tools/ncu_lines.py export.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = None
agg = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or not r[0].isdigit() or r[2] != "-":
        continue
    try:
        w, e = float(r[4]), float(r[7])
    except ValueError:
        continue
    agg[(cur, int(r[0]))] = (w, e, r[1].strip()[:90])
tot = sum(v[0] for v in agg.values())
tote = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% samples {v[1] / tote * 100:5.1f}% instrs  {k[0]}:{k[1]}  {v[2]}")
