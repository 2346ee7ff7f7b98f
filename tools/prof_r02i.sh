#!/bin/bash
# parity with the new sweep defaults, then C5 / C3 variants of the polling
# (PSCU_FLOW_POLL) and pipelined fold (PSCU_LEVEL_FOLD)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_errors.py tests/test_gpu_parity.py tests/test_gpu_3d.py -x -q > gpurun_out/t13.log 2>&1
echo "rc=$?" >> gpurun_out/t13.log
V="PSCU_FLOW_POLL=1 PSCU_LEVEL_FOLD=1;PSCU_FLOW_POLL=0 PSCU_LEVEL_FOLD=1;PSCU_FLOW_POLL=1 PSCU_LEVEL_FOLD=0;PSCU_FLOW_POLL=0 PSCU_LEVEL_FOLD=0;PSCU_FLOW_POLL=1 PSCU_LEVEL_FOLD=1 PSCU_LEVEL_FLOW_OVERSUB=1;PSCU_FLOW_POLL=1 PSCU_LEVEL_FOLD=1 PSCU_LEVEL_FLOW_OVERSUB=2"
VARIANTS="$V" SMOOTH=2 REPS=0 timeout 1200 python tools/run3d.py 64 0.1 4 5 > gpurun_out/sweep8.log 2>&1
echo "rc=$?" >> gpurun_out/sweep8.log
VARIANTS="$V" REPS=0 timeout 600 python tools/run3d.py 32 > gpurun_out/sweep9.log 2>&1
echo "rc=$?" >> gpurun_out/sweep9.log
