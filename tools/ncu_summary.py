"""Per-kernel summary of an ncu report (duration, DRAM/L2 throughput, occupancy, stalls).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy",
        "Registers Per Thread", "Compute (SM) Throughput", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ik, iname, igrid, imet, iunit, ival = (h.index(x) for x in
                                       ("ID", "Kernel Name", "Grid Size", "Metric Name",
                                        "Metric Unit", "Metric Value"))
cur = None
for r in rows[1:]:
    if len(r) <= ival:
        continue
    if r[ik] != cur:
        cur = r[ik]
        print(f"\n[{r[ik]}] {r[iname][:60]} grid {r[igrid]}")
    if r[imet] in WANT:
        print(f"    {r[imet]:36s} {r[ival]:>12s} {r[iunit]}")
