#!/bin/bash
# Full GPU check of the round's final state: test suite, smoke, default bench (config 5), reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r03g_gpu.txt
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r03g_suite.log 2>&1; echo "rc=$?" >> gpurun_out/r03g_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r03g_smoke.log
timeout 1200 python bench.py > gpurun_out/r03g_bench.json 2> gpurun_out/r03g_bench.err; echo "rc=$?" >> gpurun_out/r03g_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r03g_ref.json 2> gpurun_out/r03g_ref.err; echo "rc=$?" >> gpurun_out/r03g_ref.err
