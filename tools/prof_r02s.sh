#!/bin/bash
# Shuffle-fed backward fold (PSCU_FLOW_BSHFL) on one B200: FP64 peak probe,
# the 3D parity tests, then configs 3 and 5 with the fold off / on.
mkdir -p gpurun_out
./tools/probe_dmma > gpurun_out/r02s_probe_dmma.log 2>&1
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_zslab.py -x -q -m gpu > gpurun_out/r02s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_tests.log
SMOOTH=3 REPS=1 VARIANTS="PSCU_FLOW_BSHFL=0;PSCU_FLOW_BSHFL=1;PSCU_FLOW_BSHFL=0;PSCU_FLOW_BSHFL=1" timeout 900 python tools/run3d.py 32 0.15 1 2 > gpurun_out/r02s_c3.log 2>&1
SMOOTH=2 REPS=1 VARIANTS="PSCU_FLOW_BSHFL=0;PSCU_FLOW_BSHFL=1" timeout 1500 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r02s_c5.log 2>&1
SMOOTH=2 REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:condense_bsr -s 2 -c 1 \
   -o gpurun_out/r02s_condense python tools/run3d.py 16 0.1 4 5 > gpurun_out/r02s_ncu_condense.log 2>&1
