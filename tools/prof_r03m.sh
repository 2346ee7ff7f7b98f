#!/bin/bash
mkdir -p gpurun_out /tmp/ft
timeout 1500 python -m pytest tests/test_gpu_3d.py tests/test_gpu_zslab.py -x -q -m gpu > gpurun_out/r03m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r03m_tests.log
PSCU_LIB=tools/libpstokes_trace.so PSCU_FLOW_TRACE=/tmp/ft/ft23 PSCU_FLOW_TRACE_APPLY=50 REPS=1 \
  timeout 600 python tools/run3d.py 32 > gpurun_out/ft23_run.log 2>&1
python tools/analyze_flow_trace.py /tmp/ft/ft23_fwd.bin /tmp/ft/ft23_bwd.bin > gpurun_out/ft23_summary.txt 2>&1
rm -rf /tmp/ft
for lib in paper_2009_13840_b200/libpstokes_b200.so tools/libpstokes_b4.so; do
echo "== $lib" >> gpurun_out/r03m.log
PSCU_LIB=$lib SMOOTH=3 REPS=2 timeout 900 python tools/run3d.py 32 0.15 1 2 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); c=d['classes'].get('ilu0_apply',{})
    print('c3 solve', round(d['solve_ms'],1), 'ilu/apply', round(c['ms']/c['n'],3), 'its', d['its'], d['coarse_its'], d['rel'])
" >> gpurun_out/r03m.log
PSCU_LIB=$lib SMOOTH=2 REPS=2 timeout 1800 python tools/run3d.py 64 0.1 4 5 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); c=d['classes'].get('ilu0_apply',{})
    print('c5 solve', round(d['solve_ms'],1), 'ilu/apply', round(c['ms']/c['n'],3), 'its', d['its'], d['coarse_its'], d['rel'])
" >> gpurun_out/r03m.log
done
