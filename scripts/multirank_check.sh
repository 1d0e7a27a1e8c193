#!/bin/bash
# The multi-rank bench path on a one-GPU box: every rank on GPU 0, gloo exchange
# (FALCON_BENCH_ONE_GPU=1).  Checks that torchrun launches produce one JSON line from rank 0.
mkdir -p gpurun_out
for N in 2 4; do
  FALCON_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
    bench.py --gpus $N --workload cfg2 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/mr_cfg2_$N.json 2> gpurun_out/mr_cfg2_$N.err
  echo "cfg2 N=$N rc=$?"; tail -c 400 gpurun_out/mr_cfg2_$N.json; tail -2 gpurun_out/mr_cfg2_$N.err
done
FALCON_BENCH_ONE_GPU=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 \
  bench.py --gpus 2 --workload cfg5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/mr_cfg5_2.json 2> gpurun_out/mr_cfg5_2.err
echo "cfg5 N=2 rc=$?"; tail -c 400 gpurun_out/mr_cfg5_2.json; tail -2 gpurun_out/mr_cfg5_2.err
FALCON_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 \
  bench.py --gpus 2 --impl reference --steps 1 --warmup 1 > gpurun_out/mr_ref_2.json 2> gpurun_out/mr_ref_2.err
echo "ref N=2 rc=$?"; tail -c 300 gpurun_out/mr_ref_2.json
