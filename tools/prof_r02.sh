# Round-2 measurement batch (one GPU): default bench (config 5), then the
# ncu launch list and full captures of the 3D kernels on config 3.
set -x
python bench.py --steps 2 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file gpurun_out/launches_c3.csv python tools/run3d.py 32 > gpurun_out/ncu_c3_list.log 2>&1
for k in spmv_bsr_kernel bj_apply_kernel level_flow_kernel arnoldi_step_kernel condense_bsr_kernel resid_restrict_bsr_kernel; do
  REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 \
     -o gpurun_out/c3_$k python tools/run3d.py 32 > gpurun_out/ncu_c3_$k.log 2>&1
done
