#!/bin/bash
mkdir -p gpurun_out
V="PSCU_LEVEL_FLOW_OVERSUB=2;PSCU_LEVEL_FLOW_OVERSUB=1;PSCU_LEVEL_FLOW_OVERSUB=1.5;PSCU_LEVEL_FLOW_OVERSUB=3;PSCU_LEVEL_FLOW_OVERSUB=4;PSCU_LEVEL_FLOW_OVERSUB=2"
SMOOTH=2 REPS=0 VARIANTS="$V" timeout 1800 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r03p_c5.log 2>&1
SMOOTH=3 REPS=0 VARIANTS="$V" timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r03p_c3.log 2>&1
