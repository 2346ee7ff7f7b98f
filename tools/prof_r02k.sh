#!/bin/bash
# dataflow-sweep traces with fold cycles and the lane-parallel flag (configs 3
# and 5); analysed on the box (the raw traces exceed the copy-back limit)
mkdir -p gpurun_out /tmp/ft
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft7 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft7_run.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft7_fwd.bin /tmp/ft/ft7_bwd.bin > gpurun_out/ft7_summary.txt 2>&1
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft8 PSCU_FLOW_TRACE_APPLY=50 REPS=1 SMOOTH=2 \
  timeout 900 python tools/run3d.py 64 0.1 4 5 > gpurun_out/ft8_run.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft8_fwd.bin /tmp/ft/ft8_bwd.bin > gpurun_out/ft8_summary.txt 2>&1
rm -rf /tmp/ft
