#!/usr/bin/env python
"""Executed warp-instructions per SASS opcode from an ncu report's source page."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
c = collections.Counter(); tot = 0
rd = csv.reader(io.StringIO(out))
for r in rd:
    if len(r) < 8 or not r[0].startswith("0x"):
        continue
    ins = r[1].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    op = ins.split()[0].rstrip(";")
    base = op.split(".")[0]
    n = int(r[5])
    c[op if len(sys.argv) > 2 else base] += n; tot += n
print(f"total {tot:,}")
for op, n in c.most_common(40):
    print(f"{op:20s} {n:14,} {100*n/tot:5.1f}%")
