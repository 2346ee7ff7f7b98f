#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_3d.py -x -q -m gpu > gpurun_out/r03i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r03i_tests.log
