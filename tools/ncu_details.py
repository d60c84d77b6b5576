"""Key metrics of an ncu --set full report: python tools/ncu_details.py report.ncu-rep"""
import csv
import subprocess
import sys

WANT = ["Duration", "Memory Throughput", "DRAM Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active", "Issue Slots Busy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size", "Waves Per SM", "No Eligible",
        "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(l for l in out.splitlines() if l.startswith('"')))
hdr = rows[0]
ni, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
seen = set()
for r in rows[1:]:
    if r[ni] in WANT and r[ni] not in seen:
        seen.add(r[ni])
        print(f"{r[ni]:32s} {r[vi]:>12s} {r[ui]}")
