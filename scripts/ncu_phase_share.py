#!/usr/bin/env python
"""Stall-sample share by source-line range of one kernel file (ncu source page CSV from
`ncu -i rep --page source --csv --print-source cuda,sass`).

  ncu_phase_share.py <source.csv> <file.cuh> name:lo-hi [name:lo-hi ...]
Samples in other files (inlined helpers) are reported per file."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
target = sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    name, span = spec.split(":")
    lo, hi = span.split("-")
    ranges.append((name, int(lo), int(hi)))
path, hdr = None, None
acc, other, tot = defaultdict(int), defaultdict(int), 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and len(r) > 6 and r[2] == "-":
        try:
            n = int(r[4])
        except ValueError:
            continue
        tot += n
        if path != target:
            other[path] += n
            continue
        line = int(r[0])
        for name, lo, hi in ranges:
            if lo <= line <= hi:
                acc[name] += n
                break
        else:
            acc["(rest of " + target + ")"] += n
for k, v in list(acc.items()) + list(other.items()):
    print(f"{100.0 * v / max(tot, 1):5.1f}%  {k}")
