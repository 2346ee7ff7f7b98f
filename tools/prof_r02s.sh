#!/bin/bash
# Shuffle-fed backward fold (PSCU_FLOW_BSHFL) on one B200: FP64 peak probe,
# the 3D parity tests, then configs 3 and 5 with the fold off / on.
mkdir -p gpurun_out
./tools/probe_dmma > gpurun_out/r02s_probe_dmma.log 2>&1
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_zslab.py -x -q -m gpu > gpurun_out/r02s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_tests.log
SMOOTH=3 REPS=1 VARIANTS="PSCU_FLOW_BSHFL=0;PSCU_FLOW_BSHFL=1;PSCU_FLOW_BSHFL=0;PSCU_FLOW_BSHFL=1" timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r02s_c3.log 2>&1
PSCU_DEBUG=1 PSCU_PLAN_DEBUG=1 SMOOTH=2 REPS=1 VARIANTS="PSCU_FLOW_BSHFL=0;PSCU_FLOW_BSHFL=1" timeout 1500 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r02s_c5.log 2>&1
SMOOTH=2 REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:condense_bsr -s 2 -c 1 \
   -o gpurun_out/r02s_condense python tools/run3d.py 16 0.1 4 5 > gpurun_out/r02s_ncu_condense.log 2>&1
mkdir -p /tmp/ft
for b in 0 1; do
PSCU_FLOW_BSHFL=$b PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft12_$b PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft12_run_$b.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft12_${b}_fwd.bin /tmp/ft/ft12_${b}_bwd.bin > gpurun_out/ft12_summary_$b.txt 2>&1
done
rm -rf /tmp/ft
timeout 600 python -m pytest tests/test_gpu_3d.py -x -q -m gpu -k dmma > gpurun_out/r02s_dmma_test.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_dmma_test.log
for d in 0 1; do PSCU_CONDENSE_DMMA=$d SMOOTH=2 REPS=1 timeout 600 python tools/run3d.py 32 0.1 4 5 2>&1 | head -1 >> gpurun_out/r02s_condense_time.log; done
SMOOTH=2 REPS=1 PSCU_CONDENSE_DMMA=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:condense_bsr -s 2 -c 1 \
   -o gpurun_out/r02s_condense_dmma python tools/run3d.py 16 0.1 4 5 > gpurun_out/r02s_ncu_condense_dmma.log 2>&1
