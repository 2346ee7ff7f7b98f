#!/bin/bash
# Source-level ncu captures of the dataflow sweep kernels (config 3).
mkdir -p gpurun_out
SMOOTH=3 REPS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:level_flow_small -s 40 -c 2 \
   -o gpurun_out/r02u_flow_small python tools/run3d.py 32 0.15 1 2 > gpurun_out/r02u_ncu_flow.log 2>&1
