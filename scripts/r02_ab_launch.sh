#!/bin/bash
# A/B bench (kernel times) against AB_LIBS + per-launch ncu durations of our kernels (cfg2, cfg3).
set -u
mkdir -p gpurun_out
TESTS=${TESTS:-0} LAUNCHES=0 bash scripts/r02_iter.sh
for W in ${WORKLOADS:-cfg2 cfg3}; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_$W.csv \
    python bench.py --workload $W --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
  python - $W <<'PY'
import csv, sys
for r in csv.reader(open(f'gpurun_out/launches_{sys.argv[1]}.csv')):
    if len(r) > 14 and r[0].isdigit() and 'fb200' in r[4] and int(r[0]) > 6: print(sys.argv[1], r[4].split('(')[0][-40:], r[14])
PY
done
