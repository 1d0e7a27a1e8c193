#!/bin/bash
# Every bench line of the round (run under gpurun): cfg1..cfg5 with e2e + cpu_baseline, the
# reference arm on cfg2, and the cfg2 ncu launch list.  Output: gpurun_out/full_*.
set -u
mkdir -p gpurun_out
for W in cfg1 cfg2 cfg3; do
  timeout 1200 python bench.py --workload $W --steps 20 --warmup 5 > gpurun_out/full_$W.json 2> gpurun_out/full_$W.err
  echo "$W rc=$?"; tail -c 400 gpurun_out/full_$W.json
done
timeout 1500 python bench.py --workload cfg4 --steps 10 --warmup 3 > gpurun_out/full_cfg4.json 2> gpurun_out/full_cfg4.err; echo "cfg4 rc=$?"
timeout 1500 python bench.py --workload cfg5 --steps 5 --warmup 3 > gpurun_out/full_cfg5.json 2> gpurun_out/full_cfg5.err; echo "cfg5 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/full_ref_cfg2.json 2> gpurun_out/full_ref_cfg2.err; echo "ref rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg2.csv \
  python bench.py --workload cfg2 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "launches=$?"
