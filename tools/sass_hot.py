#!/usr/bin/env python
"""Hottest SASS lines (warp-stall samples) of an `ncu --page source --csv --print-source sass`
export, with a few lines of context: python tools/sass_hot.py <sass.csv> [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Source" in r][0]
h, body = rows[hi], rows[hi + 1:]
iS, iW = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
tot = sum(float(r[iW] or 0) for r in body) or 1.0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total samples {tot:.0f}, instructions {sum(float(r[iE] or 0) for r in body):.0f}")
for r in sorted(body, key=lambda r: -float(r[iW] or 0))[:n]:
    print(f"{float(r[iW]) / tot * 100:6.2f}%  {r[iS][:110]}")
