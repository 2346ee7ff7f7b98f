#!/bin/bash
mkdir -p gpurun_out /tmp/ft
timeout 1500 python -m pytest tests/test_gpu_3d.py tests/test_gpu_zslab.py -x -q -m gpu > gpurun_out/r03n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r03n_tests.log
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft24 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft24_run.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft24_fwd.bin /tmp/ft/ft24_bwd.bin > gpurun_out/ft24_summary.txt 2>&1
rm -rf /tmp/ft
SMOOTH=3 REPS=2 timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r03n_c3.log 2>&1
SMOOTH=2 REPS=2 timeout 1800 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r03n_c5.log 2>&1
