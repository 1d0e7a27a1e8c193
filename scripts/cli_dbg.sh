mkdir -p gpurun_out
FALCON_WALK_SPLIT=1 timeout 120 tools/bin/falcon bench --kind outlier --count 2000000 --period 100 --device --reps 3 > gpurun_out/cli_dbg.log 2>&1; echo "split rc=$?" >> gpurun_out/cli_dbg.log
FALCON_WALK_SPLIT=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 tools/bin/falcon bench --kind outlier --count 2000000 --period 100 --device --reps 3 >> gpurun_out/cli_dbg.log 2>&1; echo "split blocking rc=$?" >> gpurun_out/cli_dbg.log
timeout 120 tools/bin/falcon bench --kind outlier --count 2000000 --period 100 --device --reps 3 >> gpurun_out/cli_dbg.log 2>&1; echo "serial rc=$?" >> gpurun_out/cli_dbg.log
FALCON_WALK_SPLIT=1 timeout 200 compute-sanitizer --tool memcheck tools/bin/falcon bench --kind outlier --count 2000000 --period 100 --device --reps 1 >> gpurun_out/cli_dbg.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/cli_dbg.log
cat gpurun_out/cli_dbg.log | tail -30
