# Round-2 batch d: batched source polls in the dataflow sweeps; bitwise
# product pipeline against the config-2 fixtures.
python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_pipeline.py tests/test_gpu_c2_fixtures.py -x -q > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
REPS=1 timeout 300 python tools/run3d.py 32 > gpurun_out/r3d_32c.log 2>&1
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=gpurun_out/ft2 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft2_run.log 2>&1
SMOOTH=2 REPS=1 timeout 1500 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r3d_64c.log 2>&1
