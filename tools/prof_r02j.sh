#!/bin/bash
# shared-memory Arnoldi step: parity, then config 5 with it on / off; a
# dataflow-sweep trace of the small-task kernel at config 5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "smem or gmres or fgmres" > gpurun_out/t14.log 2>&1
echo "rc=$?" >> gpurun_out/t14.log
SMOOTH=2 REPS=1 timeout 900 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r3d_64_smem1.log 2>&1
PSCU_MGS_SMEM=0 SMOOTH=2 REPS=1 timeout 900 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r3d_64_smem0.log 2>&1
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=gpurun_out/ft6 PSCU_FLOW_TRACE_APPLY=50 REPS=1 SMOOTH=2 \
  timeout 900 python tools/run3d.py 64 0.1 4 5 > gpurun_out/ft6_run.log 2>&1
