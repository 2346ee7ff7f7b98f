#!/bin/bash
mkdir -p gpurun_out /tmp/ft
PSCU_FLOW_BSHFL=1 PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft14 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft14_run.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft14_fwd.bin /tmp/ft/ft14_bwd.bin > gpurun_out/ft14_summary.txt 2>&1
rm -rf /tmp/ft
for d in 0 1; do PSCU_CONDENSE_DMMA=$d SMOOTH=2 REPS=1 timeout 600 python tools/run3d.py 32 0.1 4 5 2>&1 | head -1 >> gpurun_out/r02v_condense_time.log; done
timeout 600 python -m pytest tests/test_gpu_3d.py -x -q -m gpu > gpurun_out/r02v_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_tests.log
