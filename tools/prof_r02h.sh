#!/bin/bash
# parity of the changed paths, the fold probe, then C5 (64^3) ILU apply:
# small-task dataflow kernel (7 CTAs/SM) x warp oversubscription, one assembly,
# one solve per variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_errors.py tests/test_gpu_parity.py tests/test_gpu_3d.py -x -q > gpurun_out/t12.log 2>&1
echo "rc=$?" >> gpurun_out/t12.log
./tools/probe_fold3 > gpurun_out/probe_fold3.log 2>&1
VARIANTS="PSCU_LEVEL_FLOW_SMALL=0 PSCU_LEVEL_FLOW_OVERSUB=1;PSCU_LEVEL_FLOW_SMALL=1 PSCU_LEVEL_FLOW_OVERSUB=1;PSCU_LEVEL_FLOW_SMALL=1 PSCU_LEVEL_FLOW_OVERSUB=2;PSCU_LEVEL_FLOW_SMALL=1 PSCU_LEVEL_FLOW_OVERSUB=3;PSCU_LEVEL_FLOW_SMALL=0 PSCU_LEVEL_FLOW_OVERSUB=2" \
  SMOOTH=2 REPS=0 timeout 1200 python tools/run3d.py 64 0.1 4 5 > gpurun_out/sweep6.log 2>&1
echo "rc=$?" >> gpurun_out/sweep6.log
VARIANTS="PSCU_LEVEL_FLOW_SMALL=0 PSCU_LEVEL_FLOW_OVERSUB=1;PSCU_LEVEL_FLOW_SMALL=1 PSCU_LEVEL_FLOW_OVERSUB=2;PSCU_LEVEL_FLOW_SMALL=1 PSCU_LEVEL_FLOW_OVERSUB=3" \
  REPS=0 timeout 600 python tools/run3d.py 32 > gpurun_out/sweep7.log 2>&1
echo "rc=$?" >> gpurun_out/sweep7.log
