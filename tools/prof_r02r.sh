#!/bin/bash
# Config 4 (3D DG, 80x80 element blocks) on one B200: GPU tests, the bench
# line at full size, the ncu launch list and full captures of the top kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dg3.py -x -q -m gpu > gpurun_out/r02r_dg3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_dg3_tests.log
timeout 1500 python bench.py --config config4 --steps 1 --warmup 3 > gpurun_out/r02r_bench_c4.json 2> gpurun_out/r02r_bench_c4.err; echo "rc=$?" >> gpurun_out/r02r_bench_c4.err
timeout 900 python bench.py --config config4 --impl reference --steps 3 --warmup 3 > gpurun_out/r02r_ref_c4.json 2> gpurun_out/r02r_ref_c4.err; echo "rc=$?" >> gpurun_out/r02r_ref_c4.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
   --log-file gpurun_out/launches_c4.csv python bench.py --config config4 --n 16 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c4_list.log 2>&1
for k in dgb_rows_kernel bj_apply_kernel arnoldi; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 10 -c 2 \
     -o gpurun_out/c4_$k python bench.py --config config4 --n 16 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c4_$k.log 2>&1
done
