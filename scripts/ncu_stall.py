#!/usr/bin/env python
"""Source lines ranked by one stall reason: python scripts/ncu_stall.py rep.ncu-rep long_sb [top]"""
import csv, io, subprocess, sys
rep, reason = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, col, tot = [], None, None, 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]; continue
    if r[0] == "Line No":
        col = r.index("stall_" + reason); continue
    if r[0] in ("Function Name", "") or col is None:
        continue
    try:
        v = int(r[col])
    except ValueError:
        continue
    tot += v
    rows.append((v, f"{fname}:{r[0]}", r[1].strip()[:80]))
rows.sort(reverse=True)
print(f"total {reason} samples {tot}")
for v, loc, src in rows[:top]:
    print(f"{100*v/max(tot,1):5.1f}% {loc:24s} {src}")
