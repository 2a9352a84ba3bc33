"""Key metrics of an ncu report (details page) — SOL, memory, scheduler, launch."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
keep = {"Duration", "DRAM Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "L2 Hit Rate",
        "Memory Throughput", "Issue Slots Busy", "Registers Per Thread", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Eligible Warps Per Scheduler", "No Eligible", "L1/TEX Hit Rate",
        "Max Bandwidth", "Mem Busy"}
seen = set()
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in keep and (d["Kernel Name"][:30], d["Metric Name"]) not in seen:
        seen.add((d["Kernel Name"][:30], d["Metric Name"]))
        print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:32s} {d['Metric Value']:>12s} {d['Metric Unit']}")
