#!/bin/bash
# Full GPU test suite + smoke on the box (logs under gpurun_out/).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${1:-suite}.log 2>&1
echo "rc=$?" >> gpurun_out/${1:-suite}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${1:-suite}_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/${1:-suite}_smoke.log
