set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "mgs_variants or plan_variants" > gpurun_out/pytest_r3.log 2>&1; tail -3 gpurun_out/pytest_r3.log
timeout 600 python tools/probe_gmres.py 256 > gpurun_out/probe_gmres_tma.log 2>&1; tail -1 gpurun_out/probe_gmres_tma.log
PSCU_MGS_TMA=0 timeout 600 python tools/probe_gmres.py 256 > gpurun_out/probe_gmres_notma.log 2>&1; tail -1 gpurun_out/probe_gmres_notma.log
timeout 900 ncu --set full --import-source on -k regex:level_kernel -s 300 -c 1 -o gpurun_out/level_k3 python tools/probe_ilu.py 256 2 0 > gpurun_out/ncu_level.log 2>&1; tail -2 gpurun_out/ncu_level.log
timeout 900 ncu --set full --import-source on -k regex:arnoldi_tma -s 200 -c 1 -o gpurun_out/arnoldi_tma python tools/probe_gmres.py 256 > gpurun_out/ncu_arn_tma.log 2>&1; tail -2 gpurun_out/ncu_arn_tma.log
