#!/usr/bin/env python
"""Stall samples and executed instructions by source line (ncu source-page CSV, gzip ok).
  ncu_lines.py <src.csv[.gz]> [N]"""
import csv
import gzip
import io
import sys
from collections import defaultdict

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fh = io.TextIOWrapper(gzip.open(path), errors="replace") if path.endswith(".gz") else open(path, errors="replace")
hdr = line = fname = None
samp, ex = defaultdict(int), defaultdict(int)
for r in csv.reader(fh):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0].isdigit():
        line = (fname, int(r[0]), r[1].strip()[:80])
    if len(r) > 7 and r[2].startswith("0x"):
        try:
            e, s = int(r[7] or 0), int(r[4] or 0)
        except ValueError:
            continue
        ex[line] += e
        samp[line] += s
ts, te = sum(samp.values()) or 1, sum(ex.values()) or 1
for k, v in sorted(samp.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100 * v / ts:5.1f}% samples {100 * ex[k] / te:5.1f}% instr  {k[0]}:{k[1]}  {k[2]}")
