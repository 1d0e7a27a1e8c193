#!/bin/bash
# Baseline of the current build on one box: GPU tests, cfg2/cfg3 bench lines, cfg2 launch list.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_gpu.log
for W in cfg2 cfg3; do
  timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "$W rc=$?"
  tail -1 gpurun_out/bench_$W.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], 'comp', r['compress_ms'], 'dec', r['decompress_ms'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --workload cfg2 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu=$?"
