#!/bin/bash
# A/B timing of library variants on the same GPU box (run under gpurun):
#   bash scripts/ab.sh WORKLOAD LIB_A LIB_B [...]   (paths relative to the repo root)
# Each variant runs the bench twice, interleaved, kernel times only.
set -u
W=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for L in "$@"; do
    FALCON_B200_LIB=$PWD/$L timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$L', 'enc_ms', round(r['encode_kernel_ms'],4), 'dec_ms', round(r['decode_kernel_ms'],4), 'step_ms', round(d['ms_per_step'],4))"
  done
done
