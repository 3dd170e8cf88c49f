"""Summarise an ncu --set full report (ncu -i ... --page details --csv) into key metrics per kernel.
    python tools/ncu_summary.py report.ncu-rep [out.txt]"""
import csv, io, subprocess, sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Issued Ipc Active",
        "Warp Cycles Per Issued Instruction", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Executed Instructions", "Compute (SM) Throughput", "No Eligible", "Block Limit Registers",
        "Block Limit Shared Mem", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ci = {x: i for i, x in enumerate(h)}
lines, cur = [], None
for r in rows[1:]:
    k = r[ci["ID"]] + " " + r[ci["Kernel Name"]][:90]
    if k != cur:
        lines.append(k)
        cur = k
    if r[ci["Metric Name"]] in WANT:
        lines.append(f"    {r[ci['Metric Name']]:40s} {r[ci['Metric Value']]:>14s} {r[ci['Metric Unit']]}")
txt = "\n".join(lines)
print(txt)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(txt + "\n")
