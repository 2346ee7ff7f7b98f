#!/bin/bash
mkdir -p gpurun_out /tmp/ft
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_zslab.py tests/test_gpu_dg3.py -x -q -m gpu > gpurun_out/r03f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r03f_tests.log
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft20 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft20_run.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft20_fwd.bin /tmp/ft/ft20_bwd.bin > gpurun_out/ft20_summary.txt 2>&1
rm -rf /tmp/ft
V="PSCU_FLOW_BFAST=0;PSCU_FLOW_BFAST=1"
SMOOTH=3 REPS=0 VARIANTS="$V" timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r03f_c3.log 2>&1
SMOOTH=2 REPS=0 VARIANTS="$V" timeout 1800 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r03f_c5.log 2>&1
