#!/bin/bash
# One build->measure iteration (run under gpurun): GPU tests, A/B bench lines, ncu captures.
#   AB="ENV=.. ENV2=.."  extra env settings to A/B against the default (cfg2 + cfg3)
#   NCU=1                ncu --set full of the encode + decode kernels (cfg2), source view
#   TESTS=0              skip pytest
set -u
mkdir -p gpurun_out
summ() { python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
    print('$1', round(d['value'],1), 'comp', round(r['compress_ms'],4), 'dec', round(r['decompress_ms'],4), 'step', round(d['ms_per_step'],4))
except Exception as e: print('$1 failed', e)"; }
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -5 gpurun_out/pytest_gpu.log
fi
for W in ${WORKLOADS:-cfg2 cfg3}; do
  for rep in 1 2; do
    timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu 2>gpurun_out/bench_err.log | summ "$W default"
    for E in ${AB:-}; do env $E timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/bench_err.log | summ "$W $E"; done
    for L in ${AB_LIBS:-}; do FALCON_B200_LIB=$PWD/$L timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/bench_err.log | summ "$W lib=$L"; done
  done
done
if [ "${LAUNCHES:-1}" = 1 ]; then
  for W in cfg2 cfg3; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_$W.csv \
      python bench.py --workload $W --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "launches $W=$?"
  done
fi
if [ "${NCU:-0}" = 1 ]; then
  for k in ${KERNELS:-encode_chunks_kernel decode_chunks_kernel}; do
    timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${NCU_W:-cfg2}_${k} -f \
      python bench.py --workload ${NCU_W:-cfg2} --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_${k}.log 2>&1
    echo "ncu $k=$?"
  done
fi
