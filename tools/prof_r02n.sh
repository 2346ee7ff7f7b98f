#!/bin/bash
mkdir -p gpurun_out /tmp/ft
timeout 120 ./tools/probe_hop 20000 > gpurun_out/probe_hop.log 2>&1
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft10 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft10_run.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft10_fwd.bin /tmp/ft/ft10_bwd.bin > gpurun_out/ft10_summary.txt 2>&1
rm -rf /tmp/ft
