#!/bin/bash
# Profiling recipe (run under gpurun, one GPU).  Writes into gpurun_out/.
#   launches.csv : every kernel launch with its device time (ncu, cold-cache, serialised)
#   prof_*.ncu-rep : one --set full capture of the encode and decode kernels
set -u
W=${1:-cfg2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_${W}.csv \
    python bench.py --workload $W --steps 3 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench_${W}.log 2>&1
for k in encode_chunks_kernel decode_chunks_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_${W}_${k} -f \
      python bench.py --workload $W --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_${W}_${k}.log 2>&1
done
