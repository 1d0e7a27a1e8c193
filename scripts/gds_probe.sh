#!/bin/bash
# Does cuFile work on this box?  (bounded: a hang is killed)
mkdir -p gpurun_out
timeout 60 python -c "
import ctypes; l=ctypes.CDLL('libcufile.so.0'); print('dlopen ok'); r=l.cuFileDriverOpen(); print('driver_open', r)" > gpurun_out/gds_probe.log 2>&1; echo "probe=$?" >> gpurun_out/gds_probe.log
timeout 120 env FALCON_CUFILE=1 python -m pytest tests/test_gpu_multi.py -k gds -x -q >> gpurun_out/gds_probe.log 2>&1; echo "cufile_test=$?" >> gpurun_out/gds_probe.log
timeout 120 python -m pytest tests/test_gpu_multi.py -k gds -x -q >> gpurun_out/gds_probe.log 2>&1; echo "bounce_test=$?" >> gpurun_out/gds_probe.log
tail -20 gpurun_out/gds_probe.log
