# cfg4 (8 GiB host-resident) and cfg5 (64 GiB sharded field, N=1) bench lines + cfg2 launch list
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
free -g | head -2; nproc
ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
for W in cfg4 cfg5; do
  timeout 1200 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
  echo "$W rc=$?"; tail -c 2500 gpurun_out/bench_$W.json; tail -3 gpurun_out/bench_$W.err
done
