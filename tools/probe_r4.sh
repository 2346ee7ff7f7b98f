set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mgs_variants or plan_variants or gmres or ilu0" > gpurun_out/pytest_r4.log 2>&1; tail -3 gpurun_out/pytest_r4.log
timeout 600 python tools/probe_ilu.py 256 20 > gpurun_out/probe_r4.log 2>&1; grep -E "level|setup" gpurun_out/probe_r4.log | tail -5
PSCU_LEVEL_CHAIN_ROWS=8 timeout 600 python tools/probe_ilu.py 256 20 0,1,2 > gpurun_out/probe_r4_g8.log 2>&1; grep -E "level" gpurun_out/probe_r4_g8.log | tail -3
PSCU_CHAIN_ROWS=3 timeout 600 python tools/probe_gmres.py 256 > gpurun_out/probe_gmres_r4.log 2>&1; tail -1 gpurun_out/probe_gmres_r4.log
PSCU_CHAIN_ROWS=3 PSCU_MGS_TMA=0 timeout 600 python tools/probe_gmres.py 256 > gpurun_out/probe_gmres_r4b.log 2>&1; tail -1 gpurun_out/probe_gmres_r4b.log
