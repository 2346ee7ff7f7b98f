#!/bin/bash
# fold restructure (row analysis: trailing / leading in-task terms) + device
# local-block producer: parity, then configs 3 and 5
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_local3.py tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_zslab.py -x -q > gpurun_out/t16.log 2>&1
echo "rc=$?" >> gpurun_out/t16.log
REPS=1 timeout 600 python tools/run3d.py 32 > gpurun_out/r3d_32_fold.log 2>&1
SMOOTH=2 REPS=1 timeout 900 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r3d_64_fold.log 2>&1
