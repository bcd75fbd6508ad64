#!/usr/bin/env python
"""Summarise ncu artefacts into small committed files under profiles/.

  ncu_summary.py report <file.ncu-rep> <out.json>   key metrics of each profiled kernel
  ncu_summary.py launches <launches.csv> <out.json> per-kernel share of a launch list
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__sass_inst_executed_op_shared_ld.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic",
]


def report(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        stalls = {}
        for i, n in enumerate(hdr):
            m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", n)
            if m and not n.endswith("not_issued"):
                try:
                    stalls[m.group(1)] = float(r[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_share_pct"] = {k: round(100 * v / tot, 1)
                                for k, v in sorted(stalls.items(), key=lambda t: -t[1])[:8]}
        res.append(d)
    json.dump({"source": path, "kernels": res}, open(out, "w"), indent=1)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    res = [{"kernel": k[:120], "launches": len(v), "avg_ns": sum(v) / len(v),
            "share_pct": round(100 * sum(v) / tot, 2)}
           for k, v in sorted(agg.items(), key=lambda t: -sum(t[1]))]
    json.dump({"source": path, "metric": "gpu__time_duration.sum (cold, serialised)",
               "kernels": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
