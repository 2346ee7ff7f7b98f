# Round-end measurement: bench line, reference arm, ncu launch list of the
# bench command (stopped once the listed launches are profiled), and full
# captures of the dominant kernels (coarse push walker, fine task-level
# kernel, Arnoldi step).
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -3 gpurun_out/ref.err; cat gpurun_out/ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 3000 --kill on --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
ncu --set full --import-source on -k regex:push_kernel -s 2 -c 1 -o gpurun_out/push_coarse python tools/probe_ilu.py 256 1 3 > gpurun_out/ncu_push.log 2>&1; tail -2 gpurun_out/ncu_push.log
ncu --set full --import-source on -k regex:level_persist -s 1 -c 1 -o gpurun_out/level_fine python tools/probe_ilu.py 256 1 0 > gpurun_out/ncu_level.log 2>&1; tail -2 gpurun_out/ncu_level.log
ncu --set full --import-source on -k regex:arnoldi -s 200 -c 1 -o gpurun_out/arnoldi_coarse python tools/probe_gmres.py 256 > gpurun_out/ncu_arn.log 2>&1; tail -2 gpurun_out/ncu_arn.log
