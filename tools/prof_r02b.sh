# Round-2 batch b: dataflow variants on config 3, parity incl. the C2
# fixtures, one full ncu capture of the config-5 coarse sweeps (traffic).
python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_c2_fixtures.py -x -q > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log
bash tools/sweep_ilu3d.sh
REPS=1 SMOOTH=2 timeout 1500 ncu --set full --clock-control none -k regex:level_flow_kernel -s 200 -c 2 \
   -o gpurun_out/c5_level_flow python tools/run3d.py 64 0.1 4 5 > gpurun_out/ncu_c5_flow.log 2>&1
