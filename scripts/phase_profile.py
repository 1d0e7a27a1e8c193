"""Aggregate ncu source-page metrics of encode/decode kernels by phase.

Phases are delimited by the '// ---- <name>' comments in the .cu source; lines of
included headers (dpds.cuh, falcon_common.cuh) count toward the phase of the call site
only approximately, so they are reported per file.
usage: python scripts/phase_profile.py <report.ncu-rep> <kernel regex> <src.cu> <values>
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre, srcfile, nvals = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
src = open(srcfile).read().split("\n")
phase_of = {}
cur = "prologue"
for i, line in enumerate(src, 1):
    m = re.search(r"// ---- ([a-z0-9 ,:\-]+)", line)
    if m:
        cur = m.group(1).strip()[:40]
    phase_of[i] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
f = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0])
target = srcfile.split("/")[-1]
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or not r or r[0] in ("", "Function Name"):
        continue
    try:
        ln = int(r[0]); ie = int(r[7] or 0); smp = int(r[4] or 0)
    except ValueError:
        continue
    key = phase_of.get(ln, "?") if f == target else "[" + f + "]"
    agg[key][0] += ie
    agg[key][1] += smp
ti = sum(a[0] for a in agg.values()) or 1
ts = sum(a[1] for a in agg.values()) or 1
print(f"{'phase':42s} {'samples%':>9s} {'instr%':>7s} {'thr-instr/value':>16s}")
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:42s} {100 * s / ts:8.1f}% {100 * i / ti:6.1f}% {i * 32 / nvals:16.1f}")
