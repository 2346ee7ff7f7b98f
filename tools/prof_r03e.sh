#!/bin/bash
mkdir -p gpurun_out /tmp/ft
./tools/probe_fp64 > gpurun_out/r03e_probe_fp64.log 2>&1
timeout 600 python -m pytest tests/test_gpu_3d.py -x -q -m gpu > gpurun_out/r03e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r03e_tests.log
SMOOTH=3 REPS=2 timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r03e_c3.log 2>&1
SMOOTH=3 REPS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:level_flow_small -s 40 -c 2 \
   -o gpurun_out/r03e_flow python tools/run3d.py 32 0.15 1 2 > gpurun_out/r03e_ncu_flow.log 2>&1
