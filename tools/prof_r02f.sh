# config-5 dataflow sweep trace (coarse level, 3.2 M rows)
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=gpurun_out/ft5 PSCU_FLOW_TRACE_APPLY=50 REPS=1 SMOOTH=2 \
  timeout 1500 python tools/run3d.py 64 0.1 4 5 > gpurun_out/ft5_run.log 2>&1
