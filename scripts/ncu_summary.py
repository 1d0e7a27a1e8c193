#!/usr/bin/env python
"""Key speed-of-light numbers of an ncu report (details page)."""
import csv, io, subprocess, sys
WANT = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Limit Registers",
        "Block Limit Shared Mem", "Dynamic Shared Memory Per Block"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]; mi = h.index("Metric Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
    print("==", rep)
    seen = set()
    for x in r[1:]:
        if x[mi] in WANT and x[mi] not in seen:
            seen.add(x[mi]); print(f"  {x[mi]:36s} {x[vi]} {x[ui]}")
