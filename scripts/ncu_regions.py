#!/usr/bin/env python
"""Aggregate an ncu source page (cuda,sass view) into per-line totals, then into
regions given as FILE:FIRST-LAST=name arguments.  Usage:
    python scripts/ncu_regions.py rep.ncu-rep encode.cu:134-160=load ..."""
import csv, io, subprocess, sys
rep = sys.argv[1]
regs = []
for a in sys.argv[2:]:
    loc, name = a.split("=")
    f, rng = loc.split(":")
    lo, hi = rng.split("-")
    regs.append((f, int(lo), int(hi), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, tot, tots, fname = {}, 0, 0, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]; continue
    if r[0] in ("Function Name", "Line No", ""):
        continue
    try:
        s, i, ln = int(r[4]), int(r[7]), int(r[0])
    except ValueError:
        continue
    tot += i; tots += s
    name = next((n for f, lo, hi, n in regs if f == fname and lo <= ln <= hi), f"{fname}:other")
    a = agg.setdefault(name, [0, 0]); a[0] += i; a[1] += s
print(f"total warp-instructions {tot:,}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:24s} {100*v[0]/tot:5.1f}% inst {100*v[1]/max(tots,1):5.1f}% stall-samples")
