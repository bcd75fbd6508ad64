#!/usr/bin/env python
"""Hottest SASS instructions (warp-stall samples) with their dominant stall reasons, from
`ncu -i rep --page source --csv --print-source cuda,sass`.

  ncu_sass_hot.py <source.csv> [N]
Also prints the stall-reason totals by SASS opcode class."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr, line, out = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if not hdr:
        continue
    if r[0].isdigit():
        line = (r[0], r[1].strip()[:60])
    if len(r) > 5 and r[2] not in ("-", "", "...") and r[2].startswith("0x"):
        try:
            s = int(r[4])
        except ValueError:
            continue
        st = {hdr[k]: int(r[k] or 0) for k in range(len(hdr)) if hdr[k].startswith("stall_") and "Not" not in hdr[k]
              and r[k] not in ("", "-")}
        out[r[2]] = (s, r[3].strip(), int(r[7] or 0), st, line)
tot = sum(v[0] for v in out.values()) or 1
byop = defaultdict(lambda: defaultdict(int))
for s, ins, ex, st, ln in out.values():
    op = ins.split()[0] if not ins.startswith("@") else ins.split()[1]
    op = op.split(".")[0]
    for k, v in st.items():
        byop[op][k] += v
    byop[op]["_all"] += s
print("== by opcode (share of all samples; top reasons)")
for op, d in sorted(byop.items(), key=lambda kv: -kv[1]["_all"])[:18]:
    rs = sorted(((v, k) for k, v in d.items() if k != "_all"), reverse=True)[:3]
    print(f"{100 * d['_all'] / tot:5.1f}% {op:<10} " + "  ".join(f"{k[6:]} {100 * v / tot:.1f}" for v, k in rs))
print("== hottest instructions")
for a, (s, ins, ex, st, ln) in sorted(out.items(), key=lambda kv: -kv[1][0])[:n]:
    rs = sorted(((v, k) for k, v in st.items()), reverse=True)[:2]
    print(f"{100 * s / tot:5.2f}% {ins[:48]:<48} ex {ex:>10} " + " ".join(f"{k[6:]}:{100 * v / tot:.2f}" for v, k in rs)
          + f"  L{ln[0] if ln else '?'}")
