#!/bin/bash
mkdir -p gpurun_out
V="PSCU_FLOW_FAR_NS=0;PSCU_FLOW_FAR_NS=300;PSCU_FLOW_FAR_NS=800;PSCU_FLOW_FAR_NS=2000;PSCU_FLOW_FAR_NS=0"
SMOOTH=3 REPS=0 VARIANTS="$V" timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r03k_c3.log 2>&1
SMOOTH=2 REPS=0 VARIANTS="$V" timeout 1800 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r03k_c5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_3d.py -x -q -m gpu > gpurun_out/r03k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r03k_tests.log
