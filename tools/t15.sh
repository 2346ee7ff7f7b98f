#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_local3.py -x -q > gpurun_out/t15.log 2>&1
echo "rc=$?" >> gpurun_out/t15.log
