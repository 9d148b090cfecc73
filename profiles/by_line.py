#!/usr/bin/env python
"""Aggregate ncu warp-stall samples by CUDA source line (needs -lineinfo):
   ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
   python profiles/by_line.py src.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur, hdr = None, None
agg, why, text = collections.Counter(), collections.defaultdict(collections.Counter), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        iW = hdr.index("Warp Stall Sampling (All Samples)")
        rs = [(i, n) for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
        continue
    if hdr is None or not r[0].isdigit() or r[2] != "-":
        continue
    v = float(r[iW]) if r[iW] not in ("", "-") else 0.0
    if v <= 0:
        continue
    key = (cur, int(r[0]))
    agg[key] += v
    text[key] = r[1]
    for i, n in rs:
        try:
            why[key][n[6:]] += float(r[i])
        except ValueError:
            pass
tot = sum(agg.values()) or 1.0
for k, v in agg.most_common(n_top):
    top = ", ".join(f"{n} {c / v * 100:.0f}%" for n, c in why[k].most_common(2))
    print(f"{v / tot * 100:5.1f}%  {k[0]}:{k[1]:<4d} {text[k].strip()[:64]:64s} [{top}]")
