#!/bin/bash
# Re-entry check: GPU test suite, smoke, default bench line + reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02x_gpu.txt
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02x_suite.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02x_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_smoke.log
timeout 1200 python bench.py > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err; echo "rc=$?" >> gpurun_out/r02x_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02x_ref.json 2> gpurun_out/r02x_ref.err; echo "rc=$?" >> gpurun_out/r02x_ref.err
