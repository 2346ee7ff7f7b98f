# occupancy (4 CTAs/SM) + optional task rotation of the dataflow sweeps; coarse block SpMV
python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py -x -q > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log
for rot in 0 1; do
  PSCU_FLOW_ROTATE=$rot REPS=1 timeout 300 python tools/run3d.py 32 > gpurun_out/r3d_32_rot$rot.log 2>&1
  PSCU_FLOW_ROTATE=$rot SMOOTH=2 REPS=1 timeout 1500 python tools/run3d.py 64 0.1 4 5 > gpurun_out/r3d_64_rot$rot.log 2>&1
done
