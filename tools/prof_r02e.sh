# Round-2 batch e: rotated task-to-warp assignment in the dataflow sweeps
python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py -x -q > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
REPS=1 timeout 300 python tools/run3d.py 32 > gpurun_out/r3d_32d.log 2>&1
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=gpurun_out/ft3 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft3_run.log 2>&1
SMOOTH=2 REPS=1 timeout 1500 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r3d_64d.log 2>&1
