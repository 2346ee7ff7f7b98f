#!/bin/bash
mkdir -p gpurun_out /tmp/ft
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft11 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft11_run.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft11_fwd.bin /tmp/ft/ft11_bwd.bin > gpurun_out/ft11_summary.txt 2>&1
rm -rf /tmp/ft
