#!/bin/bash
# Round-2 final measurement batch (one GPU): bench lines (configs 5, 3, 2a and
# the reference arm), then the config-5 ncu launch list and full captures of
# the changed kernels.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err
timeout 600 python bench.py --config config3 --steps 3 --warmup 3 > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.err
timeout 900 python bench.py --config config2a --steps 1 --warmup 3 > gpurun_out/final_bench_c2a.json 2> gpurun_out/final_bench_c2a.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref_c5.json 2> gpurun_out/final_ref_c5.err
SMOOTH=2 REPS=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
   --log-file gpurun_out/launches_c5.csv python tools/run3d.py 64 0.1 4 5 > gpurun_out/ncu_c5_list.log 2>&1
for k in level_flow_small_kernel arnoldi_smem_kernel local3_kernel; do
  SMOOTH=2 REPS=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 2 \
     -o gpurun_out/c5_$k python tools/run3d.py 64 0.1 4 5 > gpurun_out/ncu_c5_$k.log 2>&1
done
