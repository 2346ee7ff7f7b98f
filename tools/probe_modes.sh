# ILU apply times per level at 256^2 under the sweep-plan modes (default:
# push walker with chains on the coarse level, task-level launches on the
# fine levels) vs the previous row-level plans; coarse GMRES(400) classes
# with the all-gather MGS reduction vs the root-CTA one.
set -x
PSCU_DEBUG=1 timeout 600 python tools/probe_ilu.py 256 20 > gpurun_out/probe_default.log 2>&1; grep -E "level|setup|walk " gpurun_out/probe_default.log | tail -24
PSCU_WALK_MODE=push1 PSCU_WALK_CLUSTER_BWD=8 timeout 600 python tools/probe_ilu.py 256 20 3 > gpurun_out/probe_c8.log 2>&1; grep -E "level" gpurun_out/probe_c8.log | tail -2
PSCU_WALK_MODE=push1 PSCU_WALK_CLUSTER=8 timeout 600 python tools/probe_ilu.py 256 20 3 > gpurun_out/probe_c88.log 2>&1; grep -E "level" gpurun_out/probe_c88.log | tail -2
PSCU_PUSH_CONSUMERS=512 timeout 600 python tools/probe_ilu.py 256 20 3 > gpurun_out/probe_c512.log 2>&1; grep -E "level" gpurun_out/probe_c512.log | tail -2
PSCU_WALK_GRAPH=0 timeout 600 python tools/probe_ilu.py 256 20 0,1,2 > gpurun_out/probe_nograph.log 2>&1; grep -E "level" gpurun_out/probe_nograph.log | tail -3
PSCU_CHAIN_ROWS=1 PSCU_WALK_MODE=walker timeout 600 python tools/probe_ilu.py 256 20 > gpurun_out/probe_rows.log 2>&1; grep -E "level|setup" gpurun_out/probe_rows.log | tail -6
timeout 600 python tools/probe_gmres.py 256 > gpurun_out/probe_gmres.log 2>&1; tail -2 gpurun_out/probe_gmres.log
PSCU_MGS_ALL=0 timeout 600 python tools/probe_gmres.py 256 > gpurun_out/probe_gmres_root.log 2>&1; tail -2 gpurun_out/probe_gmres_root.log
PSCU_LIB=tools/libpstokes_trace.so PSCU_WALK_TRACE=1 timeout 600 python tools/probe_ilu.py 256 1 3 > gpurun_out/probe_trace.log 2>&1; grep -E "walk trace" gpurun_out/probe_trace.log | head -12
