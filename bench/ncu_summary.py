#!/usr/bin/env python
"""Summarise an ncu report (--set full) of the DP kernel into a small JSON for profiles/.

    python bench/ncu_summary.py gpurun_out/r01c_k2.ncu-rep > profiles/r01_k2_ncu_summary.json

Fields: duration, DRAM bytes (traffic for bench.py's roofline.traffic), pipe
utilisation (ALU / FMA / LSU), issue activity, occupancy, stall breakdown and the
instruction mix (share of executed warp instructions per opcode).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__occupancy_limit_registers": "occ_limit_registers",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def raw(rep):
    out = subprocess.check_output([NCU, "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    hdr, units, vals = raw(rep)
    v = vals[0]
    res = {"report": rep.split("/")[-1], "kernel": v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for k, name in METRICS.items():
        if k in hdr:
            i = hdr.index(k)
            x = v[i].replace(",", "")
            try:
                x = float(x) * SCALE.get(units[i], 1)
            except ValueError:
                pass
            res[name] = x
    if "dram_read" in res and "dram_write" in res:
        res["traffic_bytes"] = res["dram_read"] + res["dram_write"]
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[i])
    res["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
    src = subprocess.check_output([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    si, ie = h.index("Source"), h.index("Instructions Executed")
    mix = collections.Counter()
    for r in rows[2:]:
        if len(r) > ie and r[ie].isdigit():
            s = r[si].strip()
            op = s.split()[1] if s.startswith("@") else s.split()[0]
            mix[op] += int(r[ie])
    tot = sum(mix.values())
    res["warp_instructions"] = tot
    res["instruction_mix"] = {k: round(c / tot, 4) for k, c in mix.most_common(12)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
