#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_3d.py -x -q -m gpu --durations=5 > gpurun_out/r03o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r03o_tests.log
