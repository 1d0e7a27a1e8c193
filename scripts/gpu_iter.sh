#!/bin/bash
# One build->measure iteration on the GPU box (run under gpurun): GPU tests, a short
# bench line, and an ncu --set full capture of the codec kernels.  Output: gpurun_out/.
set -u
mkdir -p gpurun_out
W=${1:-cfg2}
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$W.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench_$W.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',round(d['value'],1),'enc_ms',round(r['encode_kernel_ms'],3),'dec_ms',round(r['decode_kernel_ms'],3),'enc_frac',round(r['encode_frac'],3),'dec_frac',round(r['decode_frac'],3),'ratio',d['config']['ratio'])" 2>&1
for k in ${KERNELS:-encode_chunks_kernel decode_chunks_kernel}; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_${W}_${k} -f \
      python bench.py --workload $W --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_${W}_${k}.log 2>&1
  echo "ncu $k=$?"
done
