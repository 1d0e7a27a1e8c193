#!/bin/bash
# One profiling version end to end (run under gpurun): ncu captures of the codec kernels,
# their summary (profiles/$TAG via save_profile.py, which refreshes ncu_traffic.json for
# bench.py's roofline.traffic), then every bench line (scripts/r02_full.sh).  The profile
# directory is copied into gpurun_out/ so it comes back.
set -u
TAG=${1:?tag}
mkdir -p gpurun_out
for k in encode_chunks_kernel decode_chunks_kernel sample_chunks_kernel; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_cfg2_${k} -f \
    python bench.py --workload cfg2 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_${k}.log 2>&1
  echo "ncu $k=$?"
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:encode_chunks_kernel -s 2 -c 1 -o gpurun_out/prof_cfg3_encode_chunks_kernel -f \
  python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_cfg3.log 2>&1; echo "ncu cfg3=$?"
python scripts/save_profile.py $TAG cfg2 > gpurun_out/save_profile.log 2>&1; echo "save=$?"
# the merge back is capped at 64 MiB: keep only the cfg2 encoder report (source view)
python scripts/ncu_regions.py gpurun_out/prof_cfg3_encode_chunks_kernel.ncu-rep > gpurun_out/cfg3_encode_regions.txt 2>&1
python scripts/ncu_lines2.py gpurun_out/prof_cfg2_decode_chunks_kernel.ncu-rep 0.5 > gpurun_out/cfg2_decode_lines.txt 2>&1
rm -f gpurun_out/prof_cfg2_decode_chunks_kernel.ncu-rep gpurun_out/prof_cfg2_sample_chunks_kernel.ncu-rep gpurun_out/prof_cfg3_encode_chunks_kernel.ncu-rep
bash scripts/r02_full.sh
mkdir -p gpurun_out/profiles_$TAG && cp -r profiles/$TAG/. gpurun_out/profiles_$TAG/ && cp profiles/ncu_traffic.json gpurun_out/profiles_$TAG/
