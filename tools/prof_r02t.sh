#!/bin/bash
# Reconverged shuffle fold + element-chain tasks (mid kernel) on one B200.
mkdir -p gpurun_out /tmp/ft
timeout 900 python -m pytest tests/test_gpu_3d.py -x -q -m gpu > gpurun_out/r02t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_tests.log
PSCU_LEVEL_CHAIN_ROWS=16 timeout 900 python -m pytest tests/test_gpu_3d.py -x -q -m gpu -k "hierarchy or assembly" > gpurun_out/r02t_tests16.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_tests16.log
V="PSCU_FLOW_BSHFL=0;PSCU_FLOW_BSHFL=1;PSCU_FLOW_BSHFL=1 PSCU_LEVEL_CHAIN_ROWS=16;PSCU_FLOW_BSHFL=0 PSCU_LEVEL_CHAIN_ROWS=16;PSCU_FLOW_BSHFL=1 PSCU_LEVEL_CHAIN_ROWS=12;PSCU_FLOW_BSHFL=1 PSCU_LEVEL_CHAIN_ROWS=8"
SMOOTH=3 REPS=1 VARIANTS="$V" timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r02t_c3.log 2>&1
SMOOTH=2 REPS=0 VARIANTS="$V" timeout 1800 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r02t_c5.log 2>&1
for v in "1 4" "1 16"; do set -- $v
PSCU_FLOW_BSHFL=$1 PSCU_LEVEL_CHAIN_ROWS=$2 PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft13_$2 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft13_run_$2.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft13_${2}_fwd.bin /tmp/ft/ft13_${2}_bwd.bin > gpurun_out/ft13_summary_$2.txt 2>&1
done
rm -rf /tmp/ft
SMOOTH=2 REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:condense_bsr -c 1 \
   -o gpurun_out/r02t_condense python tools/run3d.py 16 0.1 4 5 > gpurun_out/r02t_ncu_condense.log 2>&1
