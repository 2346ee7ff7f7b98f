# ILU apply times per level at 256^2: task-level launches (fine levels) and
# the push walker (coarse) under chain lengths; coarse GMRES(400) classes.
set -x
PSCU_DEBUG=1 timeout 600 python tools/probe_ilu.py 256 20 > gpurun_out/probe_default.log 2>&1; grep -E "level|setup" gpurun_out/probe_default.log | tail -8
for g in 4 8 32; do PSCU_LEVEL_CHAIN_ROWS=$g timeout 600 python tools/probe_ilu.py 256 20 0,1,2 > gpurun_out/probe_lg$g.log 2>&1; grep -E "level" gpurun_out/probe_lg$g.log | tail -3; done
for g in 2 3; do PSCU_CHAIN_ROWS=$g timeout 600 python tools/probe_ilu.py 256 20 3 > gpurun_out/probe_pg$g.log 2>&1; grep -E "level" gpurun_out/probe_pg$g.log | tail -1; done
PSCU_WALK_MODE=push1 PSCU_WALK_CLUSTER=8 timeout 600 python tools/probe_ilu.py 256 20 3 > gpurun_out/probe_c88.log 2>&1; grep -E "level" gpurun_out/probe_c88.log | tail -1
PSCU_PUSH_CONSUMERS=512 timeout 600 python tools/probe_ilu.py 256 20 3 > gpurun_out/probe_c512.log 2>&1; grep -E "level" gpurun_out/probe_c512.log | tail -1
PSCU_WALK_GRAPH=0 timeout 600 python tools/probe_ilu.py 256 20 0 > gpurun_out/probe_nograph.log 2>&1; grep -E "level" gpurun_out/probe_nograph.log | tail -1
timeout 600 python tools/probe_gmres.py 256 > gpurun_out/probe_gmres.log 2>&1; tail -1 gpurun_out/probe_gmres.log
PSCU_LIB=tools/libpstokes_trace.so PSCU_WALK_TRACE=1 timeout 600 python tools/probe_ilu.py 256 1 3 > gpurun_out/probe_trace.log 2>&1; grep -E "walk trace" gpurun_out/probe_trace.log | grep "rank=0" | head -4
