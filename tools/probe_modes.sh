# ILU apply times per level at 256^2 under the sweep-plan modes (default:
# push walker with chains on the coarse level, task-level launches on the
# fine levels) vs the previous row-level plans.
set -x
PSCU_DEBUG=1 python tools/probe_ilu.py 256 20 > gpurun_out/probe_default.log 2>&1; grep -E "level|setup|walk " gpurun_out/probe_default.log | tail -20
PSCU_CHAIN_ROWS=1 PSCU_WALK_MODE=walker python tools/probe_ilu.py 256 20 > gpurun_out/probe_rows.log 2>&1; grep -E "level|setup" gpurun_out/probe_rows.log | tail -6
PSCU_CHAIN_ROWS=8 python tools/probe_ilu.py 256 20 0,1,2 > gpurun_out/probe_g8.log 2>&1; grep -E "level" gpurun_out/probe_g8.log | tail -4
PSCU_CHAIN_ROWS=32 python tools/probe_ilu.py 256 20 0,1,2 > gpurun_out/probe_g32.log 2>&1; grep -E "level" gpurun_out/probe_g32.log | tail -4
python tools/probe_gmres.py 256 > gpurun_out/probe_gmres.log 2>&1; tail -2 gpurun_out/probe_gmres.log
