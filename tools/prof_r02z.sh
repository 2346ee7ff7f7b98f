#!/bin/bash
mkdir -p gpurun_out /tmp/ft
timeout 600 python -m pytest tests/test_gpu_3d.py -x -q -m gpu > gpurun_out/r02z_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_tests.log
for v in "1 0"; do set -- $v
PSCU_FLOW_BSHFL=$1 PSCU_FLOW_LEAD=$2 PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft18_$1_$2 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft18_run_$1_$2.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft18_$1_$2_fwd.bin /tmp/ft/ft18_$1_$2_bwd.bin > gpurun_out/ft18_summary_$1_$2.txt 2>&1
done
rm -rf /tmp/ft
V="PSCU_FLOW_BSHFL=0 PSCU_FLOW_LEAD=0;PSCU_FLOW_BSHFL=1 PSCU_FLOW_LEAD=0;PSCU_FLOW_BSHFL=1 PSCU_FLOW_LEAD=1;PSCU_FLOW_BSHFL=0 PSCU_FLOW_LEAD=1"
SMOOTH=3 REPS=1 VARIANTS="$V" timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r02z_c3.log 2>&1
SMOOTH=2 REPS=0 VARIANTS="$V" timeout 1800 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r02z_c5.log 2>&1
