#!/bin/bash
mkdir -p gpurun_out
PSCU_FLOW_LEAD=0 PSCU_FLOW_BSHFL=0 SMOOTH=3 REPS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:level_flow_small -s 41 -c 1 \
   -o gpurun_out/r03c_flow_bwd python tools/run3d.py 32 0.15 1 2 > gpurun_out/r03c_ncu_flow.log 2>&1
