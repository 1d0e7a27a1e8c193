#!/usr/bin/env python
"""Per-source-line warp-instruction and stall-sample totals of an ncu --set full report
(source page, cuda+sass view).  Usage: ncu_lines2.py REP [min_pct]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, tot, tots, fname, hdr = {}, 0, 0, None, None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].rsplit("/", 1)[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    try: ln = int(r[0])
    except ValueError: continue
    try:
        i, s = int(r[7] or 0), int(r[4] or 0)   # Instructions Executed (warp), stall samples (all)
    except ValueError: continue
    tot += i; tots += s
    a = agg.setdefault((fname, ln), [0, 0, r[1][:90]]); a[0] += i; a[1] += s
print(f"total warp-instructions {tot:,}  stall samples {tots:,}")
for (f, ln), (i, s, src) in sorted(agg.items()):
    if 100 * i / tot >= minp or 100 * s / max(tots, 1) >= minp:
        print(f"{f}:{ln:5d} {100*i/tot:5.1f}% {100*s/max(tots,1):5.1f}%  {src.strip()}")
