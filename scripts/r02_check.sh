# full GPU suite, then one bench line per single-GPU workload
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for W in ${WORKLOADS:-cfg1 cfg2 cfg3}; do
  timeout 900 python bench.py --workload $W --steps 20 --warmup 5 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
  echo "$W rc=$?"; tail -c 3000 gpurun_out/bench_$W.json; tail -3 gpurun_out/bench_$W.err
done
