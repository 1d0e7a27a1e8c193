#!/usr/bin/env python
"""Per-source-line instruction and stall-sample totals from an ncu report
(`ncu -i rep --page source --csv --print-source cuda,sass`).  Usage:
    python scripts/ncu_lines.py gpurun_out/prof.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname = [], None
tot_i = tot_s = 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        samples = int(r[4]); inst = int(r[7])
    except (ValueError, IndexError):
        continue
    rows.append((inst, samples, f"{fname}:{r[0]}", r[1].strip()[:90]))
    tot_i += inst; tot_s += samples
rows.sort(reverse=True)
print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
for inst, s, loc, src in rows[:top]:
    print(f"{100*inst/tot_i:5.1f}% inst {100*s/max(tot_s,1):5.1f}% smp  {loc:22s} {src}")
