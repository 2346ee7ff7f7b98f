# Round-2 batch c: dataflow sweep trace (config 3), spin back-off variants,
# config-5 SpMV capture, compute-sanitizer over the sweep / Arnoldi tests.
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=gpurun_out/ft PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft_run.log 2>&1
for ns in 0 64 256; do
  echo "== spin_ns=$ns" >> gpurun_out/sweep5.log
  PSCU_FLOW_SPIN_NS=$ns REPS=1 timeout 300 python tools/run3d.py 32 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['classes']['ilu0_apply']; print(d['solve_ms'], d['its'], d['coarse_its'], c['n'], c['ms'], c['ms']/c['n'])" >> gpurun_out/sweep5.log 2>&1
done
REPS=1 SMOOTH=2 timeout 1500 ncu --set full --clock-control none -k regex:spmv_bsr_kernel -s 3 -c 1 \
   -o gpurun_out/c5_spmv python tools/run3d.py 64 0.1 4 5 > gpurun_out/ncu_c5_spmv.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q \
   -k "plan_variants and 0 or gmres_mgs_variants or oversize" > gpurun_out/memcheck.log 2>&1; echo rc=$? >> gpurun_out/memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q \
   -k "plan_variants and 0-default-g3 or gmres_mgs_variants and 0-0-right" > gpurun_out/racecheck.log 2>&1; echo rc=$? >> gpurun_out/racecheck.log
