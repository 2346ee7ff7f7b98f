#!/bin/bash
mkdir -p gpurun_out /tmp/ft
./tools/probe_fold4 > gpurun_out/r02y_probe_fold4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_3d.py -x -q -m gpu > gpurun_out/r02y_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_tests.log
for v in "1 1" "1 0"; do set -- $v
PSCU_FLOW_BSHFL=$1 PSCU_FLOW_LEAD=$2 PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft17_$1_$2 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft17_run_$1_$2.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft17_$1_$2_fwd.bin /tmp/ft/ft17_$1_$2_bwd.bin > gpurun_out/ft17_summary_$1_$2.txt 2>&1
done
rm -rf /tmp/ft
V="PSCU_FLOW_BSHFL=0 PSCU_FLOW_LEAD=0;PSCU_FLOW_BSHFL=1 PSCU_FLOW_LEAD=0;PSCU_FLOW_BSHFL=1 PSCU_FLOW_LEAD=1"
SMOOTH=3 REPS=1 VARIANTS="$V" timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r02y_c3.log 2>&1
