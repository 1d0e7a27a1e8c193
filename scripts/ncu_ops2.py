#!/usr/bin/env python
"""Executed warp-instructions per SASS opcode of an ncu report (source page, sass view)."""
import csv, io, subprocess, sys, collections
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
ops, tot = collections.Counter(), 0
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "Address": hdr = r; continue
    if hdr is None or len(r) < 6: continue
    try: i = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError): continue
    src = r[1].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    ops[op.split(".")[0]] += i; tot += i
print(f"total {tot:,}")
for op, n in ops.most_common(40): print(f"{op:12s} {100*n/tot:5.1f}%  {n/ (262144):8.1f} per chunk")
