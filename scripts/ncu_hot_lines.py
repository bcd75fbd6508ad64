#!/usr/bin/env python
"""Top source lines by warp-stall samples from `ncu -i rep --page source --csv --print-source cuda,sass`.

  ncu_hot_lines.py <source.csv> [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out, path, hdr = [], None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and len(r) > 6 and r[2] == "-":
        try:
            out.append((int(r[4]), int(r[5]), int(r[7] or 0), f"{path}:{r[0]}", r[1][:90]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
for s, ni, ex, where, src in sorted(out, reverse=True)[:n]:
    print(f"{100.0 * s / tot:5.1f}% stall {100.0 * ni / tot:5.1f}% not-issued  inst {ex:>12}  {where:<22} {src}")
