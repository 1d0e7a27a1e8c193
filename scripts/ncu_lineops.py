#!/usr/bin/env python
"""Executed warp-instructions per (source line, SASS opcode) from an ncu report's
cuda+sass source page.  Usage: ncu_lineops.py REP FILE FIRST LAST"""
import csv, io, subprocess, sys, collections
rep, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, cur_line = None, None
per = collections.defaultdict(collections.Counter)
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].rsplit("/", 1)[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if r[0]:
        try: cur_line = int(r[0])
        except ValueError: cur_line = None
        continue
    # SASS row: r[2] address, r[3] sass text
    if cur_file != fname or cur_line is None or not (lo <= cur_line <= hi): continue
    try: n = int(r[7] or 0)
    except ValueError: continue
    t = r[3].strip().split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    per[cur_line][op.split(".")[0]] += n
for ln in sorted(per):
    tot = sum(per[ln].values())
    print(f"{ln:5d} {tot/262144:8.1f}/chunk  " + " ".join(f"{o}:{c/262144:.0f}" for o, c in per[ln].most_common(6)))
