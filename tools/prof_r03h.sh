#!/bin/bash
# Round-2 final profiles: bench lines (configs 3, 2a), config-5 ncu launch list,
# full captures of the dataflow sweep kernels and of the DMMA condensation variant.
mkdir -p gpurun_out
timeout 600 python bench.py --config config3 --steps 3 --warmup 3 > gpurun_out/r03h_bench_c3.json 2> gpurun_out/r03h_bench_c3.err
timeout 1500 python bench.py --config config2a --steps 1 --warmup 3 > gpurun_out/r03h_bench_c2a.json 2> gpurun_out/r03h_bench_c2a.err
SMOOTH=2 REPS=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
   --log-file gpurun_out/r03h_launches_c5.csv python tools/run3d.py 64 0.1 4 5 > gpurun_out/r03h_ncu_c5_list.log 2>&1
SMOOTH=2 REPS=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:level_flow_small -s 200 -c 2 \
   -o gpurun_out/r03h_c5_flow python tools/run3d.py 64 0.1 4 5 > gpurun_out/r03h_ncu_c5_flow.log 2>&1
for d in 0 1; do
PSCU_CONDENSE_DMMA=$d SMOOTH=2 REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:condense_bsr -c 1 \
   -o gpurun_out/r03h_condense_dmma$d python tools/run3d.py 16 0.1 4 5 > gpurun_out/r03h_ncu_condense_dmma$d.log 2>&1
done
